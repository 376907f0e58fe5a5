# ncu --set full of the offline-stage kernels without a capture yet: the
# importance-ordered pool permute and the fast scorer's window re-score
set -x
timeout 900 ncu --set full --clock-control none -k regex:"pool_permute" -c 1 -o gpurun_out/r2_permute \
  python bench.py --no-full --no-cpu --side-configs none --steps 1 --warmup 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"fs_rescore|fs_window|fs_combine" -c 3 -o gpurun_out/r2_fs_tail \
  python tools/scorer_fast_bench.py 1 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
