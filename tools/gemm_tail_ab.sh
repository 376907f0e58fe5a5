#!/bin/bash
# HISTORICAL: needs tools/probes/gemm_tail_split_variant.diff.txt applied (measured slower, not kept; profiles/round2_gemm_tail_ab.txt)
# A/B of the GEMM M-tail split (gemm.cu launch(): pair kernel over the full
# 256-row tiles + single-SM kernel over a <= 128-row remainder) vs one pair
# launch (CT_GEMM_TAIL=0).  Standalone fused gate/up + SwiGLU on the step's
# shapes, then the in-step config-2 p50 (graph replay) with the SM clock.
cd "$(dirname "$0")/.."
python -m pytest -q -x tests/test_gpu_gemm_swiglu.py 2>&1 | tail -1
for rep in 1 2; do
  for t in 0 1; do
    CT_GEMM_TAIL=$t python tools/gemm_swiglu_bench.py 2>/dev/null | grep -v "^#" | sed "s/^/tail=$t /"
  done
done
for cfg in ${CONFIGS:-cfg2}; do
  for rep in 1 2 3; do
    for t in 0 1; do
      CT_GEMM_TAIL=$t timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu \
        --no-full --side-configs none 2>/dev/null | tail -1 | python -c "
import sys, json
j = json.loads(sys.stdin.read())
print('$cfg', 'tail=$t', round(j['ms_per_step'], 2), 'eager', round(j['eager']['ms_per_step'], 2),
      j['clocks']['sm_mhz'], 'mlp', round(j['kernels']['mlp_gate_up_swiglu']['launch_ms'], 4))"
    done
  done
done
