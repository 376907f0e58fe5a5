# fast-scorer A/B: tools/probes/bin/lib_base.so (previous build) vs the
# current library (CT_FS_SIG=4 default, 8), then the GPU tests and a
# 320-chunk selection check of the current default
set -x
for rep in 1 2 3; do
timeout 300 python tools/scorer_fast_bench.py 9 --lib tools/probes/bin/lib_base.so | sed 's/^/base /'
timeout 300 python tools/scorer_fast_bench.py 9 | sed 's/^/sig4 /'
CT_FS_SIG=8 timeout 300 python tools/scorer_fast_bench.py 9 | sed 's/^/sig8 /'
done
timeout 600 python -m pytest -q -x tests/test_gpu_scorer_fast.py tests/test_gpu_fullsize.py 2>&1 | tail -3
timeout 900 python tools/scorer_fast_check.py --batches 16 --gauss 4 --out gpurun_out/scorer_split_check.json 2>&1 | tail -2
