source <(sed -n '/^set -u/,/^SMALL_PARITY/p' tools/sanitize.sh)
run memcheck scorer_fast 400 1 tests/test_gpu_scorer_fast.py
run racecheck scorer_fast 600 1 tests/test_gpu_scorer_fast.py -k "rejects or window or model"
run synccheck scorer_fast 400 1 tests/test_gpu_scorer_fast.py -k "window"
