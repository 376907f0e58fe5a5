#!/bin/bash
# A/B of the attention kernel's barrier waits: the in-tree library (plain
# spin) vs builds with -DCT_TC_SUSPEND_NS=<ns> (tools/probes/bin/lib_susp_<ns>.so,
# attention_tc.cu rebuilt with the try_wait suspend-time hint).  Standalone
# launch time (tools/attn_bench.py), output bit-identity, and the in-step
# config-2 p50 (bench.py) with the SM clock under load.
cd "$(dirname "$0")/.."
LIB=paper_2605_24022_b200/libcachetune_b200.so
cp $LIB /tmp/ct_base.so
ALTS=${ALTS:-"1000000 2000"}
for rep in 1 2 3; do
  python tools/attn_bench.py --iters 50 | sed 's/^/base /'
  for ns in $ALTS; do
    python tools/attn_bench.py --lib tools/probes/bin/lib_susp_$ns.so --iters 50 | sed "s/^/susp$ns /"
  done
done
python tools/attn_bench.py --dump gpurun_out/o_base.pt > /dev/null
for ns in $ALTS; do
  python tools/attn_bench.py --lib tools/probes/bin/lib_susp_$ns.so --dump gpurun_out/o_$ns.pt > /dev/null
  python -c "
import torch
a, b = torch.load('gpurun_out/o_base.pt'), torch.load('gpurun_out/o_$ns.pt')
print('susp$ns outputs bit-identical' if torch.equal(a, b) else 'susp$ns outputs DIFFER')
"
  rm -f gpurun_out/o_$ns.pt
done
rm -f gpurun_out/o_base.pt
for cfg in ${CONFIGS:-cfg2}; do
  for rep in 1 2; do
    for arm in base $ALTS; do
      if [ $arm = base ]; then cp /tmp/ct_base.so $LIB; else cp tools/probes/bin/lib_susp_$arm.so $LIB; fi
      timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu \
        --no-full --side-configs none 2>/dev/null | tail -1 | python -c "
import sys, json
j = json.loads(sys.stdin.read())
print('$cfg', 'instep', '$arm', round(j['ms_per_step'], 2), j['clocks']['sm_mhz'], round(j['roofline']['launch_ms'], 4))"
    done
  done
done
cp /tmp/ct_base.so $LIB
