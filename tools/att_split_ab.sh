# attention A/B: split rows (CT_TC_SPLIT=2, speculative max + pair vote) vs
# the default one-thread-per-row softmax, plus SM-clock timelines of both
# (tools/build_trace.sh -> tools/probes/bin/lib_trace.so)
set -x
CT_TC_SPLIT=2 timeout 600 python -m pytest -q -x tests/test_gpu_attention_tc.py 2>&1 | tail -3
CT_TC_SPLIT=2 timeout 300 python tools/attn_fuzz.py 2>&1 | tail -2
for rep in 1 2 3; do
timeout 120 python tools/attn_bench.py --iters 50 | sed 's/^/split1 /'
CT_TC_SPLIT=2 timeout 120 python tools/attn_bench.py --iters 50 | sed 's/^/split2 /'
done
CT_TC_TRACE_OUT=gpurun_out/trace_split1.txt timeout 120 python tools/attn_bench.py --lib tools/probes/bin/lib_trace.so --iters 3 > /dev/null
CT_TC_SPLIT=2 CT_TC_TRACE_OUT=gpurun_out/trace_split2.txt timeout 120 python tools/attn_bench.py --lib tools/probes/bin/lib_trace.so --iters 3 > /dev/null
python tools/trace_summary.py gpurun_out/trace_split1.txt
