// (4) selective-recompute attention, fp32 SIMT path (the 1e-5 parity mode)
// plus the optional AttentionRecord output.  Replaces ct/toymodel.py:176-183:
// S = q K^T / sqrt(D), key j masked iff j > pos(query), softmax, P V.
// Online softmax over 64-key tiles staged in shared memory; one warp owns a
// query row; GQA maps q-head h onto kv-head h / (Hq/Hkv).  The bf16 tensor-
// core path lives in attention_tc.cu.
#include "common.cuh"

#include <stdlib.h>

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

// ---------------------------------------------------------------------------
// Few-row path (split keys, "flash-decoding"): A x G <= DEC_MAXR rows, e.g.
// the last layer's first-token row once the other rows are pruned
// (prefill.run_layers).  A 32K-key scan by one CTA per kv head would leave
// 140 SMs idle; instead block (s, g) scores a KEYS-wide key split of kv head g
// for every row (thread per key), normalises locally and accumulates its
// partial P V (thread per head-dim column), writing (O_s, m_s, l_s) to the
// workspace; attention_decode_combine merges the splits in a fixed order
// (deterministic).  Same mask / exp2 convention as the tensor-core kernel.
constexpr int DEC_MAXR = 8;
constexpr int DEC_THREADS = 128;

inline int64_t decode_splits(int64_t n_ctx, int64_t Hkv) {
  int64_t s = (6 * 148 + Hkv - 1) / Hkv;          // ~6 CTAs per SM: loads in flight
  const int64_t cap = (n_ctx + 255) / 256;        // >= 256 keys per split
  if (s > cap) s = cap;
  const int64_t need = (n_ctx + 2047) / 2048;      // <= 2048 keys (shared memory)
  if (s < need) s = need;
  return s < 1 ? 1 : s;
}
inline int64_t decode_keys(int64_t n_ctx, int64_t splits) {
  return ((n_ctx + splits - 1) / splits + 31) / 32 * 32;
}
// 16-byte vectors along the head dim: D/VE chunks must tile the 128 threads
inline bool decode_ok(int64_t A, int64_t Hq, int64_t Hkv, int64_t D, int dtype,
                      const float* probs) {
  // CT_ATT_DECODE=0: the full kernels at tiny A (read once)
  static const bool off = [] {
    const char* e = getenv("CT_ATT_DECODE");
    return e && atoi(e) == 0;
  }();
  if (probs || off || A * (Hq / Hkv) > DEC_MAXR) return false;
  const int64_t ve = dtype == CT_BF16 ? 8 : 4;
  return D % ve == 0 && DEC_THREADS % (D / ve) == 0;
}
inline size_t decode_workspace(int64_t A, int64_t Hq, int64_t n_ctx, int64_t Hkv, int64_t D) {
  return (size_t)decode_splits(n_ctx, Hkv) * Hkv * A * (Hq / Hkv) * (D + 2) * sizeof(float);
}

inline bool cache_row_ok(const void* kc, const void* vc, int64_t crs, size_t esz) {
  return !(((uintptr_t)kc | (uintptr_t)vc) & 15) && (crs * (int64_t)esz) % 16 == 0;
}

template <typename T>
__device__ __forceinline__ void unpack_vec(const uint4& u, float* f);
template <>
__device__ __forceinline__ void unpack_vec<__nv_bfloat16>(const uint4& u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}
template <>
__device__ __forceinline__ void unpack_vec<float>(const uint4& u, float* f) {
  f[0] = __uint_as_float(u.x);
  f[1] = __uint_as_float(u.y);
  f[2] = __uint_as_float(u.z);
  f[3] = __uint_as_float(u.w);
}

template <typename T>
__global__ void __launch_bounds__(DEC_THREADS)
attention_decode_partial(const T* __restrict__ q, const int32_t* __restrict__ qpos, int A, int Hq,
                         const T* __restrict__ kc, const T* __restrict__ vc, int64_t n_ctx,
                         int Hkv, int D, int64_t crs, float scale_log2, int keys,
                         float* __restrict__ ws) {
  constexpr int VE = 16 / sizeof(T);  // elements per 16-byte vector
  extern __shared__ __align__(16) float dsm[];
  const int G = Hq / Hkv, R = A * G;
  const int CH = D / VE, KG = DEC_THREADS / CH;  // vector chunks per row, key groups
  float* sq = dsm;                 // [R][D] queries (f32)
  float* ss = sq + R * D;          // [R][keys] scores -> probabilities
  float* red = ss + R * keys;      // [KG][R][D] partial O of the key groups
  int* spos = reinterpret_cast<int*>(red + KG * R * D);
  const int split = blockIdx.x, g = blockIdx.y, tid = threadIdx.x;
  const int64_t k0 = (int64_t)split * keys;
  const int nk = (int)max((int64_t)0, min(n_ctx, k0 + keys) - k0);
  for (int t = tid; t < R * D; t += DEC_THREADS) {
    const int r = t / D, d = t % D;
    const int a = r / G, hj = r % G;
    sq[t] = to_f32(q[((int64_t)a * Hq + g * G + hj) * D + d]);
  }
  for (int r = tid; r < R; r += DEC_THREADS)
    spos[r] = (int)min((int64_t)qpos[r / G], n_ctx - 1);
  __syncthreads();
  // scores: one thread per key, the key row read as 16-byte vectors, 8 in flight
  for (int j = tid; j < nk; j += DEC_THREADS) {
    const uint4* krow = reinterpret_cast<const uint4*>(kc + (k0 + j) * crs + (int64_t)g * D);
    float acc[DEC_MAXR];
#pragma unroll
    for (int r = 0; r < DEC_MAXR; ++r) acc[r] = 0.f;
    for (int c0 = 0; c0 < CH; c0 += 8) {
      uint4 u[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (c0 + i < CH) u[i] = __ldg(krow + c0 + i);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (c0 + i >= CH) break;
        float f[VE];
        unpack_vec<T>(u[i], f);
        const int d0 = (c0 + i) * VE;
#pragma unroll
        for (int r = 0; r < DEC_MAXR; ++r) {
          if (r >= R) break;
#pragma unroll
          for (int e = 0; e < VE; ++e) acc[r] = fmaf(sq[r * D + d0 + e], f[e], acc[r]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < DEC_MAXR; ++r)
      if (r < R) ss[r * keys + j] = (k0 + j > spos[r]) ? -INFINITY : acc[r] * scale_log2;
  }
  __syncthreads();
  // per-row max and probabilities: warp w owns rows w, w+4, ...
  const int warp = tid / 32, lane = tid % 32;
  float* wsb = ws + ((int64_t)split * Hkv + g) * R * (D + 2);
  for (int r = warp; r < R; r += DEC_THREADS / 32) {
    float m = -INFINITY;
    for (int j = lane; j < nk; j += 32) m = fmaxf(m, ss[r * keys + j]);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float l = 0.f;
    for (int j = lane; j < nk; j += 32) {
      const float pj = m == -INFINITY ? 0.f : exp2f(ss[r * keys + j] - m);
      ss[r * keys + j] = pj;
      l += pj;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if (lane == 0) {
      wsb[r * (D + 2) + D] = m;
      wsb[r * (D + 2) + D + 1] = l;
    }
  }
  __syncthreads();
  // partial O = P V: thread (key group kg, chunk c) accumulates 16-byte
  // column chunk c over keys kg, kg + KG, ... (4 rows in flight), then the key
  // groups are summed through shared memory in a fixed order
  {
    const int c = tid % CH, kg = tid / CH;
    float o[DEC_MAXR][VE];
#pragma unroll
    for (int r = 0; r < DEC_MAXR; ++r)
#pragma unroll
      for (int e = 0; e < VE; ++e) o[r][e] = 0.f;
    const uint4* vbase = reinterpret_cast<const uint4*>(vc + k0 * crs + (int64_t)g * D) + c;
    const int64_t vstride = crs / VE;  // uint4 per key row
    for (int j0 = kg; j0 < nk; j0 += 4 * KG) {
      uint4 u[4];
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (j0 + i * KG < nk) u[i] = __ldg(vbase + (int64_t)(j0 + i * KG) * vstride);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int j = j0 + i * KG;
        if (j >= nk) break;
        float f[VE];
        unpack_vec<T>(u[i], f);
#pragma unroll
        for (int r = 0; r < DEC_MAXR; ++r) {
          if (r >= R) break;
          const float pj = ss[r * keys + j];
#pragma unroll
          for (int e = 0; e < VE; ++e) o[r][e] = fmaf(pj, f[e], o[r][e]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < DEC_MAXR; ++r) {
      if (r >= R) break;
#pragma unroll
      for (int e = 0; e < VE; ++e) red[(kg * R + r) * D + c * VE + e] = o[r][e];
    }
  }
  __syncthreads();
  for (int t = tid; t < R * D; t += DEC_THREADS) {
    float acc = 0.f;
    for (int kg = 0; kg < KG; ++kg) acc += red[kg * R * D + t];
    wsb[(t / D) * (D + 2) + t % D] = acc;
  }
}

// One block per (row, kv head), 128 threads: split maxima and weights by a
// fixed-shape block reduction, then thread-per-column weighted sums over the
// splits (coalesced along the head dim, 8 loads in flight).  Deterministic.
template <typename TO>
__global__ void __launch_bounds__(DEC_THREADS)
attention_decode_combine(const float* __restrict__ ws, int A, int Hq, int Hkv, int D, int splits,
                         TO* __restrict__ out) {
  extern __shared__ float cw[];  // [splits] weights 2^(m_s - M)
  __shared__ float red[DEC_THREADS / 32];
  const int G = Hq / Hkv, R = A * G;
  const int r = blockIdx.x, g = blockIdx.y, tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
  const int64_t stride = (int64_t)Hkv * R * (D + 2);
  const float* b0 = ws + ((int64_t)g * R + r) * (D + 2);
  float m = -INFINITY;
  for (int sp = tid; sp < splits; sp += DEC_THREADS) m = fmaxf(m, b0[sp * stride + D]);
#pragma unroll
  for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) red[warp] = m;
  __syncthreads();
  float M = red[0];
#pragma unroll
  for (int w = 1; w < DEC_THREADS / 32; ++w) M = fmaxf(M, red[w]);
  __syncthreads();
  float lsum = 0.f;
  for (int sp = tid; sp < splits; sp += DEC_THREADS) {
    const float ms = b0[sp * stride + D];
    const float w = ms == -INFINITY ? 0.f : exp2f(ms - M);
    cw[sp] = w;
    lsum += w * b0[sp * stride + D + 1];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
  if (lane == 0) red[warp] = lsum;
  __syncthreads();
  float L = 0.f;
#pragma unroll
  for (int w = 0; w < DEC_THREADS / 32; ++w) L += red[w];
  const float inv = L > 0.f ? 1.f / L : 0.f;
  const int a = r / G, hj = r % G;
  for (int d = tid; d < D; d += DEC_THREADS) {
    float acc = 0.f;
    int sp = 0;
    for (; sp + 8 <= splits; sp += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = b0[(sp + u) * stride + d];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = fmaf(cw[sp + u], v[u], acc);
    }
    for (; sp < splits; ++sp) acc = fmaf(cw[sp], b0[sp * stride + d], acc);
    out[((int64_t)a * Hq + g * G + hj) * D + d] = from_f32<TO>(acc * inv);
  }
}

template <typename T, typename TO>
int attention_decode(const void* q, const int32_t* q_pos, int64_t A, int64_t Hq, const void* kc,
                     const void* vc, int64_t n_ctx, int64_t Hkv, int64_t D, int64_t crs,
                     double scale, void* out, void* workspace, size_t workspace_bytes,
                     cudaStream_t st) {
  const int64_t splits = decode_splits(n_ctx, Hkv), keys = decode_keys(n_ctx, splits);
  const int64_t R = A * (Hq / Hkv);
  if (!workspace || workspace_bytes < decode_workspace(A, Hq, n_ctx, Hkv, D))
    return fail(CT_ERR_PARAM, "attention workspace too small (%zu < %zu bytes)", workspace_bytes,
                decode_workspace(A, Hq, n_ctx, Hkv, D));
  const int64_t KG = DEC_THREADS / (D / (16 / (int64_t)sizeof(T)));
  const size_t smem = (size_t)(R * D + R * keys + KG * R * D + R) * sizeof(float);
  if (cache_row_ok(kc, vc, crs, sizeof(T)) == false)
    return fail(CT_ERR_PARAM, "K/V caches must be 16-byte aligned with a 16-byte row stride");
  auto kp = attention_decode_partial<T>;
  CT_CUDA(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kp<<<dim3((unsigned)splits, (unsigned)Hkv), DEC_THREADS, smem, st>>>(
      (const T*)q, q_pos, (int)A, (int)Hq, (const T*)kc, (const T*)vc, n_ctx, (int)Hkv, (int)D,
      crs, (float)(scale * 1.4426950408889634), (int)keys, (float*)workspace);
  int rc = check_launch("attention_decode_partial");
  if (rc) return rc;
  // the weights array is padded to whole 16-byte vectors plus one: the
  // compiler reads the split tail with 16-byte shared loads (compute-sanitizer
  // memcheck flagged the over-read past an exact-size allocation)
  const size_t cw_bytes = (size_t)((splits + 3) / 4 * 4 + 4) * sizeof(float);
  attention_decode_combine<TO><<<dim3((unsigned)R, (unsigned)Hkv), DEC_THREADS, cw_bytes, st>>>(
      (const float*)workspace, (int)A, (int)Hq, (int)Hkv, (int)D, (int)splits, (TO*)out);
  return check_launch("attention_decode_combine");
}

int attention_tc(const void* q, const int32_t* q_pos, int64_t A, int64_t Hq, const void* k_cache,
                 const void* v_cache, int64_t n_ctx, int64_t Hkv, int64_t D,
                 int64_t cache_row_stride, double scale, void* out, int out_dtype,
                 void* workspace, size_t workspace_bytes, cudaStream_t st);
size_t attention_tc_workspace(int64_t A, int64_t Hq, int64_t n_ctx, int64_t Hkv, int64_t D);
bool tc_supported(const void* q, const void* k_cache, const void* v_cache, int64_t Hq,
                  int64_t Hkv, int64_t D, int64_t cache_row_stride);

}  // namespace ct

using namespace ct;

extern "C" size_t ct_attention_workspace_bytes(int64_t A, int64_t Hq, int64_t n_ctx, int64_t Hkv,
                                               int64_t D, int dtype) {
  if (A > 0 && Hq >= Hkv && Hkv > 0 && Hq % Hkv == 0 && D > 0 &&
      decode_ok(A, Hq, Hkv, D, dtype, nullptr))
    return decode_workspace(A, Hq, n_ctx, Hkv, D);
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
  if (decode_ok(A, Hq, Hkv, D, dtype, probs)) {
    if (dtype == CT_F32 && out_dtype == CT_F32)
      return attention_decode<float, float>(q, q_pos, A, Hq, k_cache, v_cache, n_ctx, Hkv, D,
                                            cache_row_stride, scale, out, workspace,
                                            workspace_bytes, st);
    if (dtype == CT_BF16 && out_dtype == CT_BF16)
      return attention_decode<__nv_bfloat16, __nv_bfloat16>(
          q, q_pos, A, Hq, k_cache, v_cache, n_ctx, Hkv, D, cache_row_stride, scale, out,
          workspace, workspace_bytes, st);
    if (dtype == CT_BF16)
      return attention_decode<__nv_bfloat16, float>(q, q_pos, A, Hq, k_cache, v_cache, n_ctx,
                                                    Hkv, D, cache_row_stride, scale, out,
                                                    workspace, workspace_bytes, st);
    return attention_decode<float, __nv_bfloat16>(q, q_pos, A, Hq, k_cache, v_cache, n_ctx, Hkv,
                                                  D, cache_row_stride, scale, out, workspace,
                                                  workspace_bytes, st);
  }
  // bf16 without a probability record: the tcgen05 kernel whenever its
  // preconditions hold (D = 128, GQA group | 128, 16-B aligned), else SIMT
  if (dtype == CT_BF16 && !probs &&
      tc_supported(q, k_cache, v_cache, Hq, Hkv, D, cache_row_stride))
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
