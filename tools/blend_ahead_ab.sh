#!/bin/bash
# HISTORICAL: needs tools/probes/blend_ahead_variant.diff.txt applied (the variant was measured and not kept; profiles/round2_blend_ahead_ab.md)
# In-step A/B of the blend schedule (HBM-resident pool): CT_BLEND_AHEAD=1
# (every layer's blend issued at the request's start on a side stream) vs 0
# (each layer's blend in line on the main stream).  p50 ms per request, SM MHz
# under load, and the blend's per-launch event time.
cd "$(dirname "$0")/.."
for cfg in ${CONFIGS:-cfg2 cfg3}; do
  for rep in 1 2 3; do
    for ahead in 0 1; do
      CT_BLEND_AHEAD=$ahead timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 \
        --no-cpu --no-full --side-configs none 2>/dev/null | tail -1 | python -c "
import sys, json
j = json.loads(sys.stdin.read())
print('$cfg', 'ahead=$ahead', round(j['ms_per_step'], 2), 'e2e', round(1e3 / j['e2e']['value'], 2),
      j['clocks']['sm_mhz'], 'blend', round(j['kernels']['gather_rope_blend']['launch_ms'], 4),
      'att', round(j['roofline']['launch_ms'], 4))"
    done
  done
done
