#!/usr/bin/env bash
# compute-sanitizer runs over the GPU tests that drive this repo's kernels
# (run on a GPU box: gpurun -- 'bash tools/sanitize.sh [quick]').
# memcheck / synccheck / racecheck instrument only namespace ct:: kernels;
# initcheck instruments every kernel (a filtered run cannot see the writes of
# torch's own kernels and reports their outputs as uninitialised).
# Logs: gpurun_out/sanitizer/<tool>_<name>.log.
set -u
OUT=${OUT:-gpurun_out/sanitizer}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
FILT=(--kernel-name kns=ct:: --kernel-name kns=_ZN2ct)
run() {  # tool name timeout filter(0/1) pytest-args...
  local tool=$1 name=$2 to=$3 filt=$4; shift 4
  local extra=()
  [ "$filt" = 1 ] && extra+=("${FILT[@]}")
  [ "$tool" = racecheck ] && extra+=(--racecheck-report analysis)
  echo "== $tool $name: pytest $*" > "$OUT/${tool}_${name}.log"
  timeout "$to" "$CS" --tool "$tool" "${extra[@]}" --print-limit 20 \
      --error-exitcode 99 --target-processes all \
      python -m pytest -q -p no:cacheprovider "$@" >> "$OUT/${tool}_${name}.log" 2>&1
  echo "== exit $?" >> "$OUT/${tool}_${name}.log"
  echo "$tool $name: $(grep -h 'ERROR SUMMARY' "$OUT/${tool}_${name}.log" | tail -1) $(tail -1 "$OUT/${tool}_${name}.log")"
}
SMALL_PARITY='spectral_cases or c_abi or rope_cases or fuse_cases or config1 or highband_cases or select_random or ragged'
run memcheck parity 600 1 tests/test_gpu_parity.py -k "$SMALL_PARITY"
run memcheck memkernels 300 1 tests/test_gpu_memkernels.py
run memcheck scorer_fast 300 1 tests/test_gpu_scorer_fast.py
run memcheck attention_tc 300 1 tests/test_gpu_attention_tc.py -k "matches_torch or f32_output or few_row"
run memcheck pool 300 1 tests/test_gpu_pool.py -k "plans_match or more_chunks or fetch_only or permute"
run memcheck gemm_swiglu 300 1 tests/test_gpu_gemm_swiglu.py -k "not 4992 and not 9920"
run initcheck memkernels 300 0 tests/test_gpu_memkernels.py -k "blend"
run initcheck parity 400 0 tests/test_gpu_parity.py -k "spectral_cases or rope_cases or fuse_cases or config1"
run initcheck attention_tc 300 0 tests/test_gpu_attention_tc.py -k "f32_output or few_row"
run synccheck parity 300 1 tests/test_gpu_parity.py -k "spectral_cases or fuse_cases or config1"
run synccheck attention_tc 300 1 tests/test_gpu_attention_tc.py -k "f32_output"
run racecheck scorer 400 1 tests/test_gpu_parity.py -k "spectral_cases and not big"
run racecheck scorer_fast 400 1 tests/test_gpu_scorer_fast.py -k "rejects or window"
run racecheck attention_tc 400 1 tests/test_gpu_attention_tc.py -k "f32_output"
run racecheck gemm_swiglu 300 1 tests/test_gpu_gemm_swiglu.py -k "128-64-128 or 129-512-384"
run synccheck gemm_swiglu 300 1 tests/test_gpu_gemm_swiglu.py -k "128-64-128 or 129-512-384"
exit 0
