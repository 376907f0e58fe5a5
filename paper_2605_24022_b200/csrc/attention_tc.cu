// (4) selective-recompute attention on tcgen05/TMEM (bf16 operands, fp32
// accumulation).  Placeholder until the tensor-core kernel lands.
#include "common.cuh"

namespace ct {
bool tc_enabled() { return false; }
size_t attention_tc_workspace(int64_t, int64_t, int64_t, int64_t, int64_t) { return 0; }
int attention_tc(const void*, const int32_t*, int64_t, int64_t, const void*, const void*, int64_t,
                 int64_t, int64_t, int64_t, double, void*, int, void*, size_t, cudaStream_t) {
  return fail(CT_ERR_UNSUPPORTED, "tcgen05 attention not built");
}
}  // namespace ct
