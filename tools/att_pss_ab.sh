# HISTORICAL: the variant this script selects was measured and removed from the
# product library (its knob is ignored now); results and source pointers are in
# profiles/round2_attention_probes.md
# attention A/B: default (P in TMEM, chained) vs P in shared memory with
# split rows (CT_TC_PSS=1: chain-free, two softmax warps per tile per SMSP)
set -x
CT_TC_PSS=1 timeout 300 python -m pytest -q -x tests/test_gpu_attention_tc.py 2>&1 | tail -3
CT_TC_PSS=1 timeout 300 python tools/attn_fuzz.py 2>&1 | tail -2
for rep in 1 2 3; do
timeout 120 python tools/attn_bench.py --iters 50 | sed 's/^/pp  /'
CT_TC_PSS=1 timeout 120 python tools/attn_bench.py --iters 50 | sed 's/^/pss /'
done
timeout 120 python tools/attn_bench.py --full | sed 's/^/pp  /'
CT_TC_PSS=1 timeout 120 python tools/attn_bench.py --full | sed 's/^/pss /'
