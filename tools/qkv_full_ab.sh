#!/bin/bash
# Full-recompute baseline with the fused QKV GEMM (CT_QKV_FUSED=1) vs cuBLAS +
# ct_qkv_rope_scatter (0), same box, interleaved: full TTFT ms, selective
# graph-replay ms, SM MHz (config 2, 32,832 rows in the full prefill).
cd "$(dirname "$0")/.."
for rep in 1 2 3; do
  for f in 0 1; do
    CT_QKV_FUSED=$f timeout 600 python bench.py --config cfg2 --steps 3 --warmup 3 --no-cpu \
      --side-configs none 2>/dev/null | tail -1 | python -c "
import sys, json
j = json.loads(sys.stdin.read())
print('fused=$f', 'full', round(j['full_recompute_ttft_ms'], 1), 'sel', round(j['ms_per_step'], 2),
      j['clocks']['sm_mhz'])"
  done
done
