// (4) selective-recompute attention, fp32 SIMT path (the 1e-5 parity mode)
// plus the optional AttentionRecord output.  Replaces ct/toymodel.py:176-183:
// S = q K^T / sqrt(D), key j masked iff j > pos(query), softmax, P V.
// Online softmax over 64-key tiles staged in shared memory; one warp owns a
// query row; GQA maps q-head h onto kv-head h / (Hq/Hkv).  The bf16 tensor-
// core path lives in attention_tc.cu.
#include "common.cuh"

namespace ct {

constexpr int AT_QB = 16;     // queries per CTA (4 per warp)
constexpr int AT_TK = 64;     // keys per tile
constexpr int AT_DMAX = 256;

template <typename T, typename TO>
__global__ void __launch_bounds__(128)
attention_simt_kernel(const T* __restrict__ q, const int32_t* __restrict__ qpos, int64_t A,
                      int Hq, const T* __restrict__ kc, const T* __restrict__ vc,
                      int64_t n_ctx, int Hkv, int D, int64_t crs, float scale,
                      TO* __restrict__ out, float* __restrict__ probs) {
  extern __shared__ __align__(16) float sm[];
  const int DP = D + 1;
  float* sq = sm;                       // [QB][D]
  float* sk = sq + AT_QB * D;           // [TK][D+1]
  float* sv = sk + AT_TK * DP;          // [TK][D+1]
  const int h = blockIdx.y;
  const int g = h / (Hq / Hkv);
  const int64_t a0 = (int64_t)blockIdx.x * AT_QB;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  constexpr int QPW = AT_QB / 4;
  constexpr int DPL = AT_DMAX / 32;  // dims per lane (max)

  int64_t maxpos = -1;
  for (int i = 0; i < AT_QB; ++i)
    if (a0 + i < A) maxpos = max(maxpos, (int64_t)qpos[a0 + i]);
  if (maxpos >= n_ctx) maxpos = n_ctx - 1;
  for (int t = threadIdx.x; t < AT_QB * D; t += blockDim.x) {
    const int i = t / D, d = t % D;
    sq[t] = (a0 + i < A) ? to_f32(q[((a0 + i) * Hq + h) * (int64_t)D + d]) : 0.f;
  }
  float m[QPW], l[QPW], acc[QPW][DPL];
  int64_t pos[QPW];
#pragma unroll
  for (int qi = 0; qi < QPW; ++qi) {
    m[qi] = -INFINITY;
    l[qi] = 0.f;
    const int64_t a = a0 + warp * QPW + qi;
    pos[qi] = a < A ? (int64_t)qpos[a] : -1;
#pragma unroll
    for (int e = 0; e < DPL; ++e) acc[qi][e] = 0.f;
  }
  for (int pass = 0; pass < (probs ? 2 : 1); ++pass) {
    const int64_t kend = pass == 0 ? maxpos + 1 : n_ctx;
    for (int64_t t0 = 0; t0 < kend; t0 += AT_TK) {
      __syncthreads();
      for (int t = threadIdx.x; t < AT_TK * D; t += blockDim.x) {
        const int j = t / D, d = t % D;
        const int64_t key = t0 + j;
        float kv = 0.f, vv = 0.f;
        if (key < n_ctx) {
          kv = to_f32(kc[key * crs + (int64_t)g * D + d]);
          if (pass == 0) vv = to_f32(vc[key * crs + (int64_t)g * D + d]);
        }
        sk[j * DP + d] = kv;
        sv[j * DP + d] = vv;
      }
      __syncthreads();
#pragma unroll
      for (int qi = 0; qi < QPW; ++qi) {
        if (pos[qi] < 0) continue;
        const float* qr = sq + (warp * QPW + qi) * D;
        float s[2];
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          const int j = lane + 32 * half;
          float dot = 0.f;
          for (int d = 0; d < D; ++d) dot += qr[d] * sk[j * DP + d];
          s[half] = (t0 + j <= pos[qi]) ? dot * scale : -INFINITY;
        }
        if (pass == 1) {
          float* prow = probs + ((int64_t)h * A + (a0 + warp * QPW + qi)) * n_ctx;
#pragma unroll
          for (int half = 0; half < 2; ++half) {
            const int64_t key = t0 + lane + 32 * half;
            if (key < n_ctx)
              prow[key] = (key <= pos[qi]) ? expf(s[half] - m[qi]) / l[qi] : 0.f;
          }
          continue;
        }
        float tmax = fmaxf(s[0], s[1]);
        for (int o = 16; o > 0; o >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
        if (tmax == -INFINITY) continue;  // whole tile masked for this query
        const float mnew = fmaxf(m[qi], tmax);
        const float corr = expf(m[qi] - mnew);
        float p0 = expf(s[0] - mnew), p1 = expf(s[1] - mnew);
        float psum = p0 + p1;
        for (int o = 16; o > 0; o >>= 1) psum += __shfl_xor_sync(0xffffffffu, psum, o);
        l[qi] = l[qi] * corr + psum;
        m[qi] = mnew;
#pragma unroll
        for (int e = 0; e < DPL; ++e) acc[qi][e] *= corr;
        for (int j = 0; j < AT_TK; ++j) {
          const float pj = __shfl_sync(0xffffffffu, j < 32 ? p0 : p1, j % 32);
          if (pj == 0.f) continue;
#pragma unroll
          for (int e = 0; e < DPL; ++e) {
            const int d = lane + 32 * e;
            if (d < D) acc[qi][e] += pj * sv[j * DP + d];
          }
        }
      }
    }
  }
#pragma unroll
  for (int qi = 0; qi < QPW; ++qi) {
    if (pos[qi] < 0) continue;
    const int64_t a = a0 + warp * QPW + qi;
    const float inv = 1.f / l[qi];
#pragma unroll
    for (int e = 0; e < DPL; ++e) {
      const int d = lane + 32 * e;
      if (d < D) out[(a * Hq + h) * (int64_t)D + d] = from_f32<TO>(acc[qi][e] * inv);
    }
  }
}

int attention_tc(const void* q, const int32_t* q_pos, int64_t A, int64_t Hq, const void* k_cache,
                 const void* v_cache, int64_t n_ctx, int64_t Hkv, int64_t D,
                 int64_t cache_row_stride, double scale, void* out, int out_dtype,
                 void* workspace, size_t workspace_bytes, cudaStream_t st);
size_t attention_tc_workspace(int64_t A, int64_t Hq, int64_t n_ctx, int64_t Hkv, int64_t D);
bool tc_enabled();

}  // namespace ct

using namespace ct;

extern "C" size_t ct_attention_workspace_bytes(int64_t A, int64_t Hq, int64_t n_ctx, int64_t Hkv,
                                               int64_t D, int dtype) {
  if (dtype == CT_BF16) return attention_tc_workspace(A, Hq, n_ctx, Hkv, D);
  return 0;
}

extern "C" int ct_selective_attention(const void* q, const int32_t* q_pos, int64_t A, int64_t Hq,
                                      const void* k_cache, const void* v_cache, int64_t n_ctx,
                                      int64_t Hkv, int64_t D, int64_t cache_row_stride,
                                      double scale, int dtype, void* out, int out_dtype,
                                      float* probs, void* workspace, size_t workspace_bytes,
                                      void* stream) {
  if (A < 0 || Hq < 1 || Hkv < 1 || Hq % Hkv || n_ctx < 1)
    return fail(CT_ERR_SHAPE, "attention geometry A=%lld Hq=%lld Hkv=%lld n_ctx=%lld",
                (long long)A, (long long)Hq, (long long)Hkv, (long long)n_ctx);
  if (D < 2 || D > AT_DMAX || D % 2) return fail(CT_ERR_SHAPE, "head_dim %lld", (long long)D);
  if (!valid_dtype(dtype) || !valid_dtype(out_dtype)) return fail(CT_ERR_PARAM, "dtype");
  if (A == 0) return CT_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (tc_enabled() && dtype == CT_BF16 && !probs && D == 128)
    return attention_tc(q, q_pos, A, Hq, k_cache, v_cache, n_ctx, Hkv, D, cache_row_stride, scale,
                        out, out_dtype, workspace, workspace_bytes, st);
  const size_t smem = (size_t)(AT_QB * D + 2 * AT_TK * (D + 1)) * sizeof(float);
  dim3 grid((unsigned)((A + AT_QB - 1) / AT_QB), (unsigned)Hq);
#define CT_ATT(T, TO)                                                                            \
  {                                                                                              \
    auto kern = attention_simt_kernel<T, TO>;                                                    \
    CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    kern<<<grid, 128, smem, st>>>((const T*)q, q_pos, A, (int)Hq, (const T*)k_cache,             \
                                  (const T*)v_cache, n_ctx, (int)Hkv, (int)D, cache_row_stride,  \
                                  (float)scale, (TO*)out, probs);                                \
  }
  if (dtype == CT_F32 && out_dtype == CT_F32) CT_ATT(float, float)
  else if (dtype == CT_BF16 && out_dtype == CT_BF16) CT_ATT(__nv_bfloat16, __nv_bfloat16)
  else if (dtype == CT_BF16 && out_dtype == CT_F32) CT_ATT(__nv_bfloat16, float)
  else CT_ATT(float, __nv_bfloat16)
#undef CT_ATT
  return check_launch("attention_simt_kernel");
}
