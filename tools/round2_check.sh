# one GPU call: new GPU tests of this round's changes, attention + scorer A/B
# against tools/probes/bin/lib_base.so, then the default bench line
set -x
timeout 900 python -m pytest -q -x tests/test_gpu_pool.py tests/test_gpu_tuner.py \
  tests/test_gpu_scorer_fast.py tests/test_gpu_attention_tc.py 2>&1 | tail -5
timeout 600 bash tools/att_ab.sh
for rep in 1 2; do
timeout 300 python tools/scorer_fast_bench.py 5 --lib tools/probes/bin/lib_base.so | sed 's/^/base /'
timeout 300 python tools/scorer_fast_bench.py 5 | sed 's/^/new  /'
done
timeout 300 python tools/scorer_fast_bench.py 1 --lib tools/probes/bin/lib_base.so --dump gpurun_out/s_base.pt > /dev/null
timeout 300 python tools/scorer_fast_bench.py 1 --dump gpurun_out/s_new.pt > /dev/null
python -c "
import torch
a, b = torch.load('gpurun_out/s_base.pt'), torch.load('gpurun_out/s_new.pt')
print('scorer agg/order identical:', torch.equal(a['agg'], b['agg']), torch.equal(a['order'], b['order']))
"
rm -f gpurun_out/s_base.pt gpurun_out/s_new.pt
timeout 600 python bench.py > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err
tail -3 gpurun_out/bench_r2.err
