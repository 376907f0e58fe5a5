// Transformer plumbing around the hot path: embedding gather
// (ct/toymodel.py:149), fused residual add + RMSNorm (ct/toymodel.py:88-89,
// :156, :184) and the MLP activation (ct/toymodel.py:186 ReLU; SwiGLU for the
// Llama geometry).  Plus the library's version / error / transfer helpers.
#include <algorithm>
#include <atomic>
#include <mutex>

#include "common.cuh"

namespace ct {

thread_local char g_last_error[512] = "";

// Launch evidence: kernel name -> number of successful launches since load or
// the last ct_launch_stats_reset.  Names are string literals (stable
// addresses); a new name takes the table mutex once, counting is lock-free.
namespace {
constexpr int kMaxKernels = 96;
std::atomic<const char*> g_kname[kMaxKernels];
std::atomic<long long> g_kcount[kMaxKernels];
std::atomic<int> g_knum{0};
std::mutex g_kmutex;
}  // namespace

void note_launch(const char* what) {
  const int n = g_knum.load(std::memory_order_acquire);
  for (int i = 0; i < n; ++i)
    if (g_kname[i].load(std::memory_order_relaxed) == what) {
      g_kcount[i].fetch_add(1, std::memory_order_relaxed);
      return;
    }
  std::lock_guard<std::mutex> lk(g_kmutex);
  const int m = g_knum.load(std::memory_order_relaxed);
  for (int i = 0; i < m; ++i)
    if (g_kname[i].load(std::memory_order_relaxed) == what) {
      g_kcount[i].fetch_add(1, std::memory_order_relaxed);
      return;
    }
  if (m == kMaxKernels) return;
  g_kname[m].store(what, std::memory_order_relaxed);
  g_kcount[m].store(1, std::memory_order_relaxed);
  g_knum.store(m + 1, std::memory_order_release);
}

__global__ void embedding_kernel(const float* __restrict__ table, const int32_t* __restrict__ tok,
                                 int64_t A, int64_t cols, float* __restrict__ out) {
  const int64_t total = A * cols;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = t / cols, c = t % cols;
    out[t] = table[(int64_t)tok[a] * cols + c];
  }
}

template <typename TD, typename TX>
__global__ void __launch_bounds__(256)
residual_rmsnorm_kernel(float* __restrict__ h, const TD* __restrict__ delta, int64_t cols,
                        double eps, TX* __restrict__ x) {
  const int64_t row = blockIdx.x;
  float* hr = h + row * cols;
  const TD* dr = delta ? delta + row * cols : nullptr;
  __shared__ double red[8];
  double ss = 0.0;
  for (int64_t c = threadIdx.x; c < cols; c += blockDim.x) {
    float v = hr[c];
    if (dr) {
      v += to_f32(dr[c]);
      hr[c] = v;
    }
    ss += (double)v * (double)v;
  }
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    red[0] = t;
  }
  __syncthreads();
  const float inv = (float)(1.0 / sqrt(red[0] / (double)cols + eps));
  if (x)
    for (int64_t c = threadIdx.x; c < cols; c += blockDim.x)
      x[row * cols + c] = from_f32<TX>(hr[c] * inv);
}

// Vectorised residual + RMSNorm: one CTA per row, the row held in registers
// (float4 per thread-slot), so h and delta are read once and h, x written once.
template <int VPT, typename TX, int NT = 256>
__global__ void __launch_bounds__(NT)
residual_rmsnorm_vec_kernel(float* __restrict__ h, const float* __restrict__ delta, int64_t cols,
                            double eps, TX* __restrict__ x) {
  const int64_t row = blockIdx.x;
  float4* hr = reinterpret_cast<float4*>(h + row * cols);
  const float4* dr = delta ? reinterpret_cast<const float4*>(delta + row * cols) : nullptr;
  const int nv = (int)(cols / 4);
  float4 v[VPT];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int c = threadIdx.x + i * NT;
    if (c < nv) {
      float4 a = hr[c];
      if (dr) {
        const float4 d = __ldg(dr + c);
        a.x += d.x; a.y += d.y; a.z += d.z; a.w += d.w;
        hr[c] = a;
      }
      v[i] = a;
      ss += a.x * a.x + a.y * a.y + a.z * a.z + a.w * a.w;
    }
  }
  __shared__ float red[NT / 32];
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) tot += red[w];
  const float inv = (float)(1.0 / sqrt((double)tot / (double)cols + eps));
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int c = threadIdx.x + i * NT;
    if (c < nv) {
      TX* xo = x + row * cols + 4 * (int64_t)c;
      if constexpr (sizeof(TX) == 2) {
        __nv_bfloat162 lo = __floats2bfloat162_rn(v[i].x * inv, v[i].y * inv);
        __nv_bfloat162 hi = __floats2bfloat162_rn(v[i].z * inv, v[i].w * inv);
        uint2 u;
        u.x = *reinterpret_cast<uint32_t*>(&lo);
        u.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(xo) = u;
      } else {
        *reinterpret_cast<float4*>(xo) = make_float4(v[i].x * inv, v[i].y * inv, v[i].z * inv,
                                                     v[i].w * inv);
      }
    }
  }
}

// RMSNorm without a residual (the residual add lives in the GEMM epilogues):
// a CTA walks rows r, r + gridDim, ... keeping the next row's h in registers
// while it reduces and stores the current one.
template <int VPT, typename TX>
__global__ void __launch_bounds__(256)
rmsnorm_rows_kernel(const float* __restrict__ h, int64_t A, double eps, TX* __restrict__ x) {
  constexpr int COLS = 4 * 256 * VPT;
  __shared__ float red[2][8];
  float4 cur[VPT], nxt[VPT];
  int64_t row = blockIdx.x;
  if (row >= A) return;
#pragma unroll
  for (int i = 0; i < VPT; ++i)
    cur[i] = ldg_stream_f4(reinterpret_cast<const float4*>(h + row * COLS) + threadIdx.x + i * 256);
  for (int par = 0; row < A; row += gridDim.x, par ^= 1) {
    const int64_t nrow = row + gridDim.x;
    if (nrow < A) {
#pragma unroll
      for (int i = 0; i < VPT; ++i)
        nxt[i] = ldg_stream_f4(reinterpret_cast<const float4*>(h + nrow * COLS) + threadIdx.x +
                               i * 256);
    }
    float ss = 0.f;
#pragma unroll
    for (int i = 0; i < VPT; ++i)
      ss += cur[i].x * cur[i].x + cur[i].y * cur[i].y + cur[i].z * cur[i].z + cur[i].w * cur[i].w;
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    if ((threadIdx.x & 31) == 0) red[par][threadIdx.x >> 5] = ss;
    __syncthreads();
    float tot = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) tot += red[par][w];
    const float inv = (float)(1.0 / sqrt((double)tot / (double)COLS + eps));
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      TX* xo = x + row * COLS + 4 * (int64_t)(threadIdx.x + i * 256);
      if constexpr (sizeof(TX) == 2) {
        __nv_bfloat162 lo = __floats2bfloat162_rn(cur[i].x * inv, cur[i].y * inv);
        __nv_bfloat162 hi = __floats2bfloat162_rn(cur[i].z * inv, cur[i].w * inv);
        uint2 u;
        u.x = *reinterpret_cast<uint32_t*>(&lo);
        u.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(xo) = u;
      } else {
        *reinterpret_cast<float4*>(xo) = make_float4(cur[i].x * inv, cur[i].y * inv,
                                                     cur[i].z * inv, cur[i].w * inv);
      }
    }
#pragma unroll
    for (int i = 0; i < VPT; ++i) cur[i] = nxt[i];
  }
}

// SwiGLU on 8-wide bf16 vectors: act = silu(gate) * up.
__global__ void swiglu_vec_kernel(const uint4* __restrict__ gu, int64_t A, int64_t inter8,
                                  uint4* __restrict__ act) {
  const int64_t total = A * inter8;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = t / inter8, i = t % inter8;
    const uint4 g = __ldg(gu + a * 2 * inter8 + i);
    const uint4 u = __ldg(gu + a * 2 * inter8 + inter8 + i);
    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&g);
    const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&u);
    uint4 o;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 gf = __bfloat1622float2(g2[k]);
      const float2 uf = __bfloat1622float2(u2[k]);
      o2[k] = __floats2bfloat162_rn(gf.x / (1.f + __expf(-gf.x)) * uf.x,
                                    gf.y / (1.f + __expf(-gf.y)) * uf.y);
    }
    act[t] = o;
  }
}

// One 16-byte group of 8 outputs per thread, rows on blockIdx.y: no 64-bit
// division per element, and enough CTAs resident that every SM keeps ~64 KB
// of gate/up loads in flight.
__device__ __forceinline__ float silu_tanh(float g) {
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * g));
  const float hg = 0.5f * g;
  return fmaf(hg, t, hg);
}

template <bool LOOP, bool TANH = true>
__global__ void __launch_bounds__(256)
swiglu_row_kernel(const uint4* __restrict__ gu, int64_t A, int64_t inter8,
                  uint4* __restrict__ act) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= inter8) return;
  // LOOP only when A exceeds one grid dimension (65535 rows)
  for (int64_t a = blockIdx.y; LOOP ? a < A : a == blockIdx.y; a += gridDim.y) {
    const uint4 g = ldg_stream(gu + a * 2 * inter8 + i);
    const uint4 u = ldg_stream(gu + a * 2 * inter8 + inter8 + i);
    const __nv_bfloat162* g2 = reinterpret_cast<const __nv_bfloat162*>(&g);
    const __nv_bfloat162* u2 = reinterpret_cast<const __nv_bfloat162*>(&u);
    uint4 o;
    __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(&o);
  #pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 gf = __bfloat1622float2(g2[k]);
      const float2 uf = __bfloat1622float2(u2[k]);
      // silu(g) = g sigmoid(g) = 0.5 g (1 + tanh(g / 2)): one MUFU op per
      // element instead of ex2 + rcp (the kernel is MUFU-co-bound at the
      // power-capped step clock); tanh.approx error ~2^-11, output is bf16
      if constexpr (TANH)
        o2[k] = __floats2bfloat162_rn(silu_tanh(gf.x) * uf.x, silu_tanh(gf.y) * uf.y);
      else
        o2[k] = __floats2bfloat162_rn(gf.x / (1.f + __expf(-gf.x)) * uf.x,
                                      gf.y / (1.f + __expf(-gf.y)) * uf.y);
    }
    act[a * inter8 + i] = o;
  }
}

static const bool g_swiglu_v1 = getenv("CT_SWIGLU_V1") != nullptr;
static const bool g_swiglu_exp = getenv("CT_SWIGLU_EXP") != nullptr;  // ex2 + rcp form

template <typename TI, typename TO>
__global__ void mlp_act_kernel(const TI* __restrict__ gu, int64_t A, int64_t inter, int kind,
                               TO* __restrict__ act) {
  const int64_t total = A * inter;
  const int64_t ld = kind == 0 ? 2 * inter : inter;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = t / inter, i = t % inter;
    const float g = to_f32(gu[a * ld + i]);
    float r;
    if (kind == 0) {
      const float u = to_f32(gu[a * ld + inter + i]);
      r = g / (1.f + expf(-g)) * u;
    } else {
      r = fmaxf(g, 0.f);
    }
    act[t] = from_f32<TO>(r);
  }
}

static unsigned grid_cap(int64_t units) {
  int64_t b = (units + 255) / 256;
  if (b > 148 * 32) b = 148 * 32;
  return (unsigned)(b < 1 ? 1 : b);
}

}  // namespace ct

using namespace ct;

extern "C" int ct_version(void) { return 1; }

extern "C" int ct_last_error(char* buf, size_t len) {
  if (!buf || !len) return CT_ERR_PARAM;
  strncpy(buf, g_last_error, len - 1);
  buf[len - 1] = 0;
  return CT_OK;
}

extern "C" int ct_launch_stats(char* buf, size_t len) {
  if (!buf || !len) return fail(CT_ERR_PARAM, "ct_launch_stats: empty buffer");
  size_t used = 0;
  buf[0] = 0;
  const int n = g_knum.load(std::memory_order_acquire);
  for (int i = 0; i < n; ++i) {
    const int w = snprintf(buf + used, len - used, "%s%s=%lld", i ? ";" : "",
                           g_kname[i].load(std::memory_order_relaxed),
                           (long long)g_kcount[i].load(std::memory_order_relaxed));
    if (w < 0 || (size_t)w >= len - used) return fail(CT_ERR_PARAM, "ct_launch_stats: buffer too small");
    used += (size_t)w;
  }
  return CT_OK;
}

extern "C" void ct_launch_stats_reset(void) {
  const int n = g_knum.load(std::memory_order_acquire);
  for (int i = 0; i < n; ++i) g_kcount[i].store(0, std::memory_order_relaxed);
}

extern "C" int ct_device_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return 0; }
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

extern "C" int ct_embedding_gather(const float* table, const int32_t* tokens, int64_t A,
                                   int64_t cols, float* out, void* stream) {
  if (A == 0) return CT_OK;
  embedding_kernel<<<grid_cap(A * cols), 256, 0, (cudaStream_t)stream>>>(table, tokens, A, cols, out);
  return check_launch("embedding_kernel");
}

static const bool g_rms_v1 = getenv("CT_RMS_V1") != nullptr;

extern "C" int ct_residual_rmsnorm(float* h, const void* delta, int delta_dtype, int64_t A,
                                   int64_t cols, double eps, void* x_out, int x_dtype,
                                   void* stream) {
  if (A == 0) return CT_OK;
  if (!valid_dtype(delta_dtype) || !valid_dtype(x_dtype)) return fail(CT_ERR_PARAM, "dtype");
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned g = (unsigned)A;
  const bool aligned = ((uintptr_t)h % 16 == 0) && ((uintptr_t)delta % 16 == 0) &&
                       ((uintptr_t)x_out % 16 == 0) && x_out != nullptr;
  // no residual, rows of 4 * 256 * VPT f32 -> x: persistent row loop with the
  // next row's loads issued before this row's reduction and stores
  if (delta == nullptr && cols == 4 * 256 * 4 && aligned && !g_rms_v1) {
    // 3..16 CTAs per SM measured flat (22.6 us for 4992 x 4096)
    const unsigned grid = (unsigned)std::min<int64_t>(A, 148 * 6);
    if (x_dtype == CT_BF16)
      rmsnorm_rows_kernel<4, __nv_bfloat16><<<grid, 256, 0, st>>>(h, A, eps, (__nv_bfloat16*)x_out);
    else
      rmsnorm_rows_kernel<4, float><<<grid, 256, 0, st>>>(h, A, eps, (float*)x_out);
    return check_launch("rmsnorm_rows_kernel");
  }
  if (delta_dtype == CT_F32 && cols % 4 == 0 && cols <= 4 * 256 * 8 && aligned) {
    const int vpt = (int)((cols / 4 + 255) / 256);
#define CT_RMS(V)                                                                                  \
  if (vpt <= V) {                                                                                  \
    if (x_dtype == CT_BF16)                                                                        \
      residual_rmsnorm_vec_kernel<V, __nv_bfloat16><<<g, 256, 0, st>>>(h, (const float*)delta,     \
                                                                       cols, eps,                  \
                                                                       (__nv_bfloat16*)x_out);     \
    else                                                                                           \
      residual_rmsnorm_vec_kernel<V, float><<<g, 256, 0, st>>>(h, (const float*)delta, cols, eps,  \
                                                               (float*)x_out);                     \
    return check_launch("residual_rmsnorm_vec_kernel");                                            \
  }
    CT_RMS(1) CT_RMS(2) CT_RMS(4) CT_RMS(8)
#undef CT_RMS
  }
  if (delta_dtype == CT_F32 && x_dtype == CT_F32)
    residual_rmsnorm_kernel<float, float><<<g, 256, 0, st>>>(h, (const float*)delta, cols, eps, (float*)x_out);
  else if (delta_dtype == CT_F32 && x_dtype == CT_BF16)
    residual_rmsnorm_kernel<float, __nv_bfloat16><<<g, 256, 0, st>>>(h, (const float*)delta, cols, eps, (__nv_bfloat16*)x_out);
  else if (delta_dtype == CT_BF16 && x_dtype == CT_BF16)
    residual_rmsnorm_kernel<__nv_bfloat16, __nv_bfloat16><<<g, 256, 0, st>>>(h, (const __nv_bfloat16*)delta, cols, eps, (__nv_bfloat16*)x_out);
  else
    residual_rmsnorm_kernel<__nv_bfloat16, float><<<g, 256, 0, st>>>(h, (const __nv_bfloat16*)delta, cols, eps, (float*)x_out);
  return check_launch("residual_rmsnorm_kernel");
}

extern "C" int ct_mlp_act(const void* gu, int64_t A, int64_t inter, int in_dtype, int kind,
                          void* act, int act_dtype, void* stream) {
  if (A == 0) return CT_OK;
  if (kind != 0 && kind != 1) return fail(CT_ERR_PARAM, "mlp kind %d", kind);
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned g = grid_cap(A * inter);
  if (kind == 0 && in_dtype == CT_BF16 && act_dtype == CT_BF16 && inter % 8 == 0 &&
      ((uintptr_t)gu % 16 == 0) && ((uintptr_t)act % 16 == 0)) {
    if (!g_swiglu_v1) {
      const int64_t inter8 = inter / 8;
      const unsigned gy = (unsigned)std::min<int64_t>(A, 65535);
      const dim3 grid((unsigned)((inter8 + 255) / 256), gy);
      if (A <= 65535 && g_swiglu_exp)
        swiglu_row_kernel<false, false><<<grid, 256, 0, st>>>((const uint4*)gu, A, inter8,
                                                              (uint4*)act);
      else if (A <= 65535)
        swiglu_row_kernel<false><<<grid, 256, 0, st>>>((const uint4*)gu, A, inter8, (uint4*)act);
      else
        swiglu_row_kernel<true><<<grid, 256, 0, st>>>((const uint4*)gu, A, inter8, (uint4*)act);
      return check_launch("swiglu_row_kernel");
    }
    swiglu_vec_kernel<<<grid_cap(A * inter / 8), 256, 0, st>>>((const uint4*)gu, A, inter / 8,
                                                                (uint4*)act);
    return check_launch("swiglu_vec_kernel");
  }
  if (in_dtype == CT_F32 && act_dtype == CT_F32)
    mlp_act_kernel<float, float><<<g, 256, 0, st>>>((const float*)gu, A, inter, kind, (float*)act);
  else if (in_dtype == CT_BF16 && act_dtype == CT_BF16)
    mlp_act_kernel<__nv_bfloat16, __nv_bfloat16><<<g, 256, 0, st>>>((const __nv_bfloat16*)gu, A, inter, kind, (__nv_bfloat16*)act);
  else if (in_dtype == CT_F32 && act_dtype == CT_BF16)
    mlp_act_kernel<float, __nv_bfloat16><<<g, 256, 0, st>>>((const float*)gu, A, inter, kind, (__nv_bfloat16*)act);
  else
    mlp_act_kernel<__nv_bfloat16, float><<<g, 256, 0, st>>>((const __nv_bfloat16*)gu, A, inter, kind, (float*)act);
  return check_launch("mlp_act_kernel");
}

extern "C" int ct_copy_ranges_h2d(void* const* dst, const void* const* src, const int64_t* bytes,
                                  int64_t n, void* stream) {
  for (int64_t i = 0; i < n; ++i) {
    if (bytes[i] <= 0) continue;
    CT_CUDA(cudaMemcpyAsync(dst[i], src[i], (size_t)bytes[i], cudaMemcpyHostToDevice,
                            (cudaStream_t)stream));
  }
  return CT_OK;
}

extern "C" int ct_host_alloc(void** ptr, size_t bytes) {
  CT_CUDA(cudaHostAlloc(ptr, bytes, cudaHostAllocDefault));
  return CT_OK;
}

extern "C" int ct_host_free(void* ptr) {
  CT_CUDA(cudaFreeHost(ptr));
  return CT_OK;
}
