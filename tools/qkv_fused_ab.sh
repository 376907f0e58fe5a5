#!/bin/bash
# In-step A/B of the fused q|k|v GEMM + RoPE/scatter epilogue
# (ct_gemm_qkv_rope, CT_QKV_FUSED=1) vs cuBLAS + ct_qkv_rope_scatter
# (CT_QKV_FUSED=0): graph-replay p50, eager p50, SM MHz, attention launch ms.
cd "$(dirname "$0")/.."
for cfg in ${CONFIGS:-cfg2 cfg3}; do
  for rep in 1 2 3; do
    for f in 0 1; do
      CT_QKV_FUSED=$f timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu \
        --no-full --side-configs none 2>/dev/null | tail -1 | python -c "
import sys, json
j = json.loads(sys.stdin.read())
k = j['kernels']
print('$cfg', 'fused=$f', round(j['ms_per_step'], 2), 'eager', round(j['eager']['ms_per_step'], 2),
      j['clocks']['sm_mhz'], 'qkv_gemm', None if not k.get('qkv_gemm_rope') else round(k['qkv_gemm_rope']['launch_ms'], 4),
      'frac', None if not k.get('qkv_gemm_rope') else round(k['qkv_gemm_rope']['frac'], 3))"
    done
  done
done
