#!/bin/bash
# A/B of the fused gate/up + SwiGLU tcgen05 GEMM (ct_gemm_swiglu) against
# cuBLAS + ct_mlp_act, end to end through bench.py (CT_MLP_FUSED=0/1),
# interleaved so clock drift hits both arms.  Prints one line per run:
# config, arm, ms_per_step, value, full-recompute TTFT ms, speed-up.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for cfg in ${CONFIGS:-cfg2 cfg3}; do
  for arm in 1 0 1 0; do
    CT_MLP_FUSED=$arm timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 \
      --no-cpu --side-configs none > gpurun_out/mlp_ab_${cfg}_${arm}.json 2>/dev/null
    python - "$cfg" "$arm" <<'PY'
import json, sys
cfg, arm = sys.argv[1:]
j = json.loads(open(f"gpurun_out/mlp_ab_{cfg}_{arm}.json").read().strip().splitlines()[-1])
print(cfg, f"fused={arm}", j["ms_per_step"], j["value"], j.get("full_recompute_ttft_ms"), j.get("ttft_speedup_vs_full"))
PY
  done
done
