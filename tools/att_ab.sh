# attention A/B: round-1 library vs current (POLY variants) + timeline trace
python -m pytest -q -x tests/test_gpu_attention_tc.py 2>&1 | tail -2
for rep in 1 2; do
python tools/attn_bench.py --lib tools/probes/bin/lib_r1.so --iters 50 | sed 's/^/r1    /'
for p in 0 1 5; do CT_TC_POLY=$p python tools/attn_bench.py --iters 50 | sed "s/^/poly$p /"; done
done
python tools/attn_bench.py --lib tools/probes/bin/lib_r1.so --full | sed 's/^/r1    /'
for p in 0 1; do CT_TC_POLY=$p python tools/attn_bench.py --full | sed "s/^/poly$p /"; done
for p in 0 1; do CT_TC_POLY=$p CT_TC_TRACE_OUT=gpurun_out/att_trace$p.txt python tools/attn_bench.py --lib tools/probes/bin/lib_trace.so --iters 3 >/dev/null; done
