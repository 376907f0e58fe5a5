// Standalone tcgen05 GEMM probe (sm_100a): C[M,N] = A[M,K] B[K,N], bf16 in,
// f32 accumulate in TMEM, bf16 out -- the MLP gate/up shape of config 2
// (M 4992, K 4096, N 28672), to see whether a hand-written kernel reaches
// cuBLAS before fusing the SwiGLU epilogue.  Optional SwiGLU epilogue
// (mode 1): the N-tile holds 128 gate + 128 up columns and the kernel writes
// act = silu(gate) * up [M, N/2].
//   warp 0: TMA producer (A box 64K x 128M, four B boxes 64N x 64K per stage)
//   warp 1: MMA issuer (M128 N256 K16, A K-major, B MN-major, SWIZZLE_128B)
//   warps 2-5: epilogue (one TMEM lane per thread, double-buffered accumulators)
// Persistent: one CTA per SM, tiles N-outer so consecutive CTAs share B in L2.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gemm_probe gemm_probe.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;          // 16 KiB
constexpr int B_BYTES = BN * BK * 2;          // 32 KiB (4 N-atoms of 64 x 64)
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t par) {
  asm volatile("{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
               "@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(b), "r"(par) : "memory");
}
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];"
               ::"r"(dst), "l"(m), "r"(bar), "r"(c0), "r"(c1) : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void commit(uint32_t b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc) : "memory");
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ void ld32(uint32_t t, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                 "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                 "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t pack(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// mode 0: C [M, N] bf16; mode 1: act [M, N/2] = silu(gate) * up, where the
// N-tile t covers gate columns [128 t, 128 t + 128) and up columns
// [N/2 + 128 t, N/2 + 128 t + 128) (the B boxes are fetched from both halves)
template <int MODE>
__global__ void __launch_bounds__(192, 1) gemm(const __grid_constant__ CUtensorMap ma,
                                               const __grid_constant__ CUtensorMap mb,
                                               __nv_bfloat16* __restrict__ out, int M, int N, int K) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t bar = base + STAGES * STAGE_BYTES;
  auto full = [&](int s) { return bar + s * 8; };
  auto empty = [&](int s) { return bar + (STAGES + s) * 8; };
  auto afull = [&](int b) { return bar + (2 * STAGES + b) * 8; };
  auto aempty = [&](int b) { return bar + (2 * STAGES + 2 + b) * 8; };
  uint32_t* tptr = reinterpret_cast<uint32_t*>(gbase + STAGES * STAGE_BYTES + (2 * STAGES + 4) * 8);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int mt = M / BM, nt = (MODE ? N / 2 / 128 : N / BN), tiles = mt * nt, kt = K / BK;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(full(s), 1); mbar_init(empty(s), 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(afull(b), 1); mbar_init(aempty(b), 128); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tptr)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tptr;
  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int n_i = t / mt, m_i = t % mt;
        for (int k = 0; k < kt; ++k) {
          mbar_wait(empty(s), ph ^ 1);
          const uint32_t st = base + s * STAGE_BYTES;
          mbar_expect_tx(full(s), STAGE_BYTES);
          tma2d(st, &ma, full(s), k * BK, m_i * BM);
          for (int i = 0; i < 4; ++i) {
            const int col = MODE ? ((i < 2 ? 0 : N / 2) + n_i * 128 + (i & 1) * 64) : n_i * BN + i * 64;
            tma2d(st + A_BYTES + i * 8192, &mb, full(s), col, k * BK);
          }
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // kind::f16, bf16 A/B, f32 D, B MN-major, N = 256, M = 128
      constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                                 ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      int s = 0, it = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
        const int b = it & 1;
        mbar_wait(aempty(b), (uint32_t)(((it >> 1) & 1) ^ 1));
        fence_after();
        const uint32_t acc = tmem + b * 256;
        for (int k = 0; k < kt; ++k) {
          mbar_wait(full(s), ph);
          fence_after();
          const uint32_t st = base + s * STAGE_BYTES;
          const uint64_t ad = sdesc(st, 16, 1024), bd = sdesc(st + A_BYTES, 8192, 1024);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            mma(acc, ad + (uint64_t)((kk * 32) >> 4), bd + (uint64_t)((kk * 2048) >> 4), IDESC, (k | kk) ? 1u : 0u);
          commit(empty(s));
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        commit(afull(b));
      }
    }
  } else {
    // epilogue: warps 2..5 -> TMEM lane quarter (warp % 4)
    const int q = warp & 3, row = q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    int it = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int b = it & 1, n_i = t / mt, m_i = t % mt;
      mbar_wait(afull(b), (uint32_t)((it >> 1) & 1));
      fence_after();
      const uint32_t acc = tmem + b * 256 + lane_off;
      const int64_t grow = (int64_t)m_i * BM + row;
      if (MODE == 0) {
        uint4* dst = reinterpret_cast<uint4*>(out + grow * N + (int64_t)n_i * BN);
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          uint32_t r[32];
          ld32(acc + c * 32, r);
#pragma unroll
          for (int e = 0; e < 4; ++e)
            dst[c * 4 + e] = make_uint4(pack(__uint_as_float(r[8 * e]), __uint_as_float(r[8 * e + 1])),
                                        pack(__uint_as_float(r[8 * e + 2]), __uint_as_float(r[8 * e + 3])),
                                        pack(__uint_as_float(r[8 * e + 4]), __uint_as_float(r[8 * e + 5])),
                                        pack(__uint_as_float(r[8 * e + 6]), __uint_as_float(r[8 * e + 7])));
        }
      } else {
        uint4* dst = reinterpret_cast<uint4*>(out + grow * (N / 2) + (int64_t)n_i * 128);
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t g[32], u[32];
          ld32(acc + c * 32, g);
          ld32(acc + 128 + c * 32, u);
          float a[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const float x = __uint_as_float(g[e]);
            a[e] = x / (1.f + __expf(-x)) * __uint_as_float(u[e]);
          }
#pragma unroll
          for (int e = 0; e < 4; ++e)
            dst[c * 4 + e] = make_uint4(pack(a[8 * e], a[8 * e + 1]), pack(a[8 * e + 2], a[8 * e + 3]),
                                        pack(a[8 * e + 4], a[8 * e + 5]), pack(a[8 * e + 6], a[8 * e + 7]));
        }
      }
      fence_before();
      mbar_arrive(aempty(b));
    }
  }
  fence_before();
  __syncthreads();
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return (PFN_cuTensorMapEncodeTiled_v12000)p;
}
static void map2d(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint32_t b0, uint32_t b1) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {inner * 2};
  cuuint32_t box[2] = {b0, b1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("tensor map failed %d\n", (int)r); exit(1); }
}

__global__ void fill(__nv_bfloat16* p, int64_t n, uint32_t seed, float scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = __float2bfloat16(((x & 0xffff) / 32768.f - 1.f) * scale);
  }
}

int main(int argc, char** argv) {
  const int M = 4992, K = 4096, N = 28672;
  __nv_bfloat16 *A, *B, *C;
  cudaMalloc(&A, (size_t)M * K * 2);
  cudaMalloc(&B, (size_t)K * N * 2);
  cudaMalloc(&C, (size_t)M * N * 2);
  fill<<<1024, 256>>>(A, (int64_t)M * K, 1, 1.f);
  fill<<<1024, 256>>>(B, (int64_t)K * N, 2, 1.f / 64.f);
  CUtensorMap ma, mb;
  map2d(&ma, A, K, M, 64, 128);   // A [M][K]: box 64 K x 128 rows
  map2d(&mb, B, N, K, 64, 64);    // B [K][N]: box 64 N x 64 K
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = STAGES * STAGE_BYTES + 1024 + 256;
  for (int mode = 0; mode < 2; ++mode) {
    auto k = mode ? gemm<1> : gemm<0>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int w = 0; w < 3; ++w) k<<<sms, 192, smem>>>(ma, mb, C, M, N, K);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    const int it = 20;
    for (int i = 0; i < it; ++i) k<<<sms, 192, smem>>>(ma, mb, C, M, N, K);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= it;
    printf("mode %d (%s): %.1f us  %.0f TFLOP/s  err=%s\n", mode, mode ? "gate/up + SwiGLU epilogue" : "plain GEMM",
           ms * 1e3, 2.0 * M * N * K / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  }
  // correctness spot check of mode 0 against a simple reference on a few entries
  gemm<0><<<sms, 192, smem>>>(ma, mb, C, M, N, K);
  cudaDeviceSynchronize();
  __nv_bfloat16* hA = (__nv_bfloat16*)malloc((size_t)M * K * 2);
  __nv_bfloat16* hB = (__nv_bfloat16*)malloc((size_t)K * N * 2);
  __nv_bfloat16* hC = (__nv_bfloat16*)malloc((size_t)M * N * 2);
  cudaMemcpy(hA, A, (size_t)M * K * 2, cudaMemcpyDeviceToHost);
  cudaMemcpy(hB, B, (size_t)K * N * 2, cudaMemcpyDeviceToHost);
  cudaMemcpy(hC, C, (size_t)M * N * 2, cudaMemcpyDeviceToHost);
  double worst = 0;
  for (int s = 0; s < 64; ++s) {
    const int i = (s * 977) % M, j = (s * 7919 + 13) % N;
    double ref = 0;
    for (int k = 0; k < K; ++k) ref += (double)__bfloat162float(hA[(size_t)i * K + k]) * __bfloat162float(hB[(size_t)k * N + j]);
    const double got = __bfloat162float(hC[(size_t)i * N + j]);
    worst = fmax(worst, fabs(got - ref) / (fabs(ref) + 1e-3));
  }
  printf("spot check: worst rel err %.3e over 64 entries\n", worst);
  return 0;
}
