# compute-sanitizer memcheck over the engine tests that drive the pinned-pool
# staging ring (copy stream + blend) and the corpus bind path
source <(sed -n '/^set -u/,/^SMALL_PARITY/p' tools/sanitize.sh)
run memcheck pool_ring 900 1 tests/test_gpu_pool.py -k "hbm_and_pinned or corpus or more_chunks"
