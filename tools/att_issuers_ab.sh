# HISTORICAL: the variant this script selects was measured and removed from the
# product library (its knob is ignored now); results and source pointers are in
# profiles/round2_attention_probes.md
# attention A/B: one MMA issuer for both tiles (default) vs one per tile
# (CT_TC_ISSUERS=2), tests + fuzzer on the new variant, SM-clock timelines
set -x
CT_TC_ISSUERS=2 timeout 600 python -m pytest -q -x tests/test_gpu_attention_tc.py 2>&1 | tail -3
CT_TC_ISSUERS=2 timeout 300 python tools/attn_fuzz.py 2>&1 | tail -2
for rep in 1 2 3; do
timeout 120 python tools/attn_bench.py --iters 50 | sed 's/^/iss1 /'
CT_TC_ISSUERS=2 timeout 120 python tools/attn_bench.py --iters 50 | sed 's/^/iss2 /'
done
timeout 120 python tools/attn_bench.py --full | sed 's/^/iss1 /'
CT_TC_ISSUERS=2 timeout 120 python tools/attn_bench.py --full | sed 's/^/iss2 /'
CT_TC_TRACE_OUT=gpurun_out/trace_iss1.txt timeout 120 python tools/attn_bench.py --lib tools/probes/bin/lib_trace.so --iters 3 > /dev/null
CT_TC_ISSUERS=2 CT_TC_TRACE_OUT=gpurun_out/trace_iss2.txt timeout 120 python tools/attn_bench.py --lib tools/probes/bin/lib_trace.so --iters 3 > /dev/null
python tools/trace_summary.py gpurun_out/trace_iss1.txt gpurun_out/trace_iss2.txt
