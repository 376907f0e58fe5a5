# attention A/B of the round-2 split-row variant (CT_TC_SPLIT=2; the kernel
# template was not committed; see profiles/round2_attention_probes.md): previous vs current library
set -x
CT_TC_SPLIT=2 timeout 600 python -m pytest -q -x tests/test_gpu_attention_tc.py 2>&1 | tail -3
CT_TC_SPLIT=2 timeout 300 python tools/attn_fuzz.py 2>&1 | tail -3
for rep in 1 2 3; do
timeout 120 python tools/attn_bench.py --lib tools/probes/bin/lib_base.so --iters 50 | sed 's/^/base   /'
timeout 120 python tools/attn_bench.py --iters 50 | sed 's/^/split1 /'
CT_TC_SPLIT=2 timeout 120 python tools/attn_bench.py --iters 50 | sed 's/^/split2 /'
done
timeout 120 python tools/attn_bench.py --full | sed 's/^/split1 /'
CT_TC_SPLIT=2 timeout 120 python tools/attn_bench.py --full | sed 's/^/split2 /'
