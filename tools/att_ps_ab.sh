# HISTORICAL: the variant this script selects was measured and removed from the
# product library (its knob is ignored now); results and source pointers are in
# profiles/round2_attention_probes.md
# attention A/B: P in TMEM (attention_pp_kernel, default) vs P in shared
# memory with S(j+1) issued once S(j) is loaded (attention_ps_kernel,
# CT_TC_PS=1), with FMA-pipe exp2 for 0 / 25 / 50 % of the keys (CT_TC_POLY)
set -x
CT_TC_PS=1 CT_TC_POLY=5 timeout 300 python -m pytest -q -x tests/test_gpu_attention_tc.py 2>&1 | tail -2
CT_TC_PS=1 CT_TC_POLY=1 timeout 300 python tools/attn_fuzz.py 2>&1 | tail -1
for rep in 1 2; do
timeout 120 python tools/attn_bench.py --iters 50 | sed 's/^/pp      /'
for pm in 0 1 4 5; do
CT_TC_PS=1 CT_TC_POLY=$pm timeout 120 python tools/attn_bench.py --iters 50 | sed "s/^/ps-poly$pm /"
done
done
timeout 120 python tools/attn_bench.py --full | sed 's/^/pp      /'
for pm in 0 1 5; do
CT_TC_PS=1 CT_TC_POLY=$pm timeout 120 python tools/attn_bench.py --full | sed "s/^/ps-poly$pm /"
done
