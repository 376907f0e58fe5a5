# attention A/B: tools/probes/bin/lib_base.so (previous build) vs the current
# library, timings interleaved, output bit-compare, timeline trace of the new
# kernel (tools/build_trace.sh -> lib_trace.so, built before the call)
python -m pytest -q -x tests/test_gpu_attention_tc.py 2>&1 | tail -2
for rep in 1 2 3; do
python tools/attn_bench.py --lib tools/probes/bin/lib_base.so --iters 50 | sed 's/^/base /'
python tools/attn_bench.py --iters 50 | sed 's/^/new  /'
CT_TC_POLY=1 python tools/attn_bench.py --iters 50 | sed 's/^/newp1 /'
CT_TC_POLY=4 python tools/attn_bench.py --iters 50 | sed 's/^/newp4 /'
done
python tools/attn_bench.py --lib tools/probes/bin/lib_base.so --full | sed 's/^/base /'
python tools/attn_bench.py --full | sed 's/^/new  /'
python tools/attn_bench.py --lib tools/probes/bin/lib_base.so --dump gpurun_out/o_base.pt > /dev/null
python tools/attn_bench.py --dump gpurun_out/o_new.pt > /dev/null
python -c "
import torch
a, b = torch.load('gpurun_out/o_base.pt'), torch.load('gpurun_out/o_new.pt')
d = (a.float() - b.float()).abs().max().item()
print('outputs bit-identical' if torch.equal(a, b) else f'outputs differ: max abs {d:.3e}')
"
rm -f gpurun_out/o_base.pt gpurun_out/o_new.pt
if [ -f tools/probes/bin/lib_trace.so ]; then
CT_TC_TRACE_OUT=gpurun_out/att_trace_new.txt python tools/attn_bench.py --lib tools/probes/bin/lib_trace.so --iters 3 > /dev/null
python tools/trace_summary.py gpurun_out/att_trace_new.txt
fi
