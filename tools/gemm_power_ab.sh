#!/bin/bash
# In-step A/B of two builds of the library: arm "base" = the in-tree
# libcachetune_b200.so, arm "alt" = tools/probes/bin/libcachetune_b200_alt.so
# (e.g. gemm.cu rebuilt with -DCT_GEMM_SUSPEND_NS=0, the plain-spin barrier
# waits; profiles/round2_gemm_power_ab.txt was measured with base = plain
# spin and alt = the 1 ms suspend hint, now the default), each with the
# QKV / O / down projections on cuBLAS (CT_GEMM_OWN=0) and on ct_gemm_bf16
# (CT_GEMM_OWN=1).
cd "$(dirname "$0")/.."
LIB=paper_2605_24022_b200/libcachetune_b200.so
cp $LIB /tmp/ct_base.so
for cfg in ${CONFIGS:-cfg2 cfg3}; do
  for rep in 1 2; do
    for arm in base alt; do
      if [ $arm = alt ]; then cp tools/probes/bin/libcachetune_b200_alt.so $LIB; else cp /tmp/ct_base.so $LIB; fi
      for own in 0 1; do
        CT_GEMM_OWN=$own timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu \
          --no-full --side-configs none 2>/dev/null | tail -1 | python -c "
import sys, json
j = json.loads(sys.stdin.read())
print('$cfg', '$arm', 'own=$own', round(j['ms_per_step'], 2), j['clocks']['sm_mhz'])"
      done
    done
  done
done
cp /tmp/ct_base.so $LIB
