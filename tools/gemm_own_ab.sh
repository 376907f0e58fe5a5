#!/bin/bash
# In-step A/B: O- and down-projections on ct_gemm_bf16 (CT_GEMM_OWN=1) vs cuBLAS (0), with the fused QKV GEMM on; graph-replay ms, eager ms, SM MHz
cd "$(dirname "$0")/.."
for cfg in cfg2 cfg3; do for rep in 1 2 3; do for own in 0 1; do
CT_GEMM_OWN=$own timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu --no-full --side-configs none 2>/dev/null | tail -1 | python -c "
import sys, json
j = json.loads(sys.stdin.read())
print('$cfg', 'own=$own', round(j['ms_per_step'], 2), 'eager', round(j['eager']['ms_per_step'], 2), j['clocks']['sm_mhz'])"
done; done; done
