// Gate/up projection with the SwiGLU activation fused into the epilogue, on
// the 5th-gen tensor cores (sm_100a).  Replaces, for the bf16 step, the pair
//     gu = x @ W_gu (cuBLAS)   ->   act = silu(gu[:, :I]) * gu[:, I:]  (ct_mlp_act)
// of ct/toymodel.py:184-186 (the SwiGLU MLP of the restated Llama/Mistral
// geometry): the [M, 2I] gate/up product never reaches HBM, and the
// activation is computed from the f32 accumulators.
//
// C tile = 128 rows x 256 accumulator columns = 128 gate + the matching 128
// up columns, so one N-tile yields 128 finished activation columns.
//   warp 0   TMA producer: per 64-deep K stage one A box (64 K x 128 rows,
//            K-major) and four B boxes (64 N x 64 K, MN-major: 2 gate + 2 up),
//            SWIZZLE_128B, a 4-stage ring (48 KiB per stage)
//   warp 1   MMA issuer: tcgen05.mma kind::f16 M128 N256 K16, f32 in TMEM
//            (+ TMEM allocation)
//   warps 2-5 epilogue: one TMEM lane (= output row) per thread,
//            silu(g) * u in f32, bf16 16-byte stores
// TMEM holds two 256-column accumulators, so the epilogue of tile t runs
// under the MMAs of tile t+1.  Persistent: one CTA per SM walks the tiles
// N-major within L2-sized bands of M-tiles (TileMap), so consecutive CTAs
// share the B tile and the A slice stays in L2.  Rows past M are zero-filled
// by TMA and not stored.
#include "common.cuh"

#include <cuda.h>
#include <algorithm>
#include <cudaTypedefs.h>

namespace ct {
namespace gm {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;          // 16 KiB
constexpr int B_BYTES = BN * BK * 2;          // 32 KiB: four 64 x 64 N-atoms
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int NBAR = 2 * STAGES + 4;
constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + NBAR * 8 + 16 + 1024;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t par) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLW:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra LD;\n\tbra LW;\n\tLD:\n\t}" ::"r"(b),
      "r"(par)
      : "memory");
}
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0,
                                      int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(m), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void commit(uint32_t b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b)
               : "memory");
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
// shared-memory matrix descriptor, SWIZZLE_128B, sm100 version bit
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
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(t));
}
// wait::ld, threading the registers through so their uses cannot move above it
__device__ __forceinline__ void ld_wait(uint32_t* r) {
  asm volatile(
      "tcgen05.wait::ld.sync.aligned;"
      : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]),
        "+r"(r[7]), "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]),
        "+r"(r[14]), "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]),
        "+r"(r[20]), "+r"(r[21]), "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]),
        "+r"(r[26]), "+r"(r[27]), "+r"(r[28]), "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
      :
      : "memory");
}
__device__ __forceinline__ uint32_t pack(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

// Tile order: bands of `band_m` M-tiles (an A slice of <= ~60 MB that stays
// in L2), N-major inside a band so consecutive CTAs share the B tile.  One
// band when A fits (config 2's 4992 rows); the 32K-row full prefill walks
// five bands instead of streaming all of A from HBM once per N-tile.
struct TileMap {
  int mt, nt, band_m;
  __device__ __forceinline__ void at(int t, int& m_i, int& n_i) const {
    const int band_full = band_m * nt, band = t / band_full, r = t - band * band_full;
    const int m_lo = band * band_m, bm = min(band_m, mt - m_lo);
    n_i = r / bm;
    m_i = m_lo + (r - n_i * bm);
  }
};

__global__ void __launch_bounds__(192, 1)
gemm_swiglu_kernel(const __grid_constant__ CUtensorMap map_x,
                   const __grid_constant__ CUtensorMap map_w, __nv_bfloat16* __restrict__ act,
                   int M, int I, int K, int64_t ld_act, int band_m) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t bar = base + STAGES * STAGE_BYTES;
  auto full = [&](int s) { return bar + s * 8; };
  auto empty = [&](int s) { return bar + (STAGES + s) * 8; };
  auto afull = [&](int b) { return bar + (2 * STAGES + b) * 8; };
  auto aempty = [&](int b) { return bar + (2 * STAGES + 2 + b) * 8; };
  uint32_t* tptr = reinterpret_cast<uint32_t*>(gbase + STAGES * STAGE_BYTES + NBAR * 8);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int mt = (M + BM - 1) / BM, nt = I / 128, tiles = mt * nt, kt = K / BK;
  const TileMap tm{mt, nt, band_m};
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full(s), 1);
      mbar_init(empty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(afull(b), 1);
      mbar_init(aempty(b), 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     su32(tptr))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tptr;
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        int m_i, n_i;
        tm.at(t, m_i, n_i);
        for (int k = 0; k < kt; ++k) {
          mbar_wait(empty(s), ph ^ 1);
          const uint32_t st = base + s * STAGE_BYTES;
          mbar_expect_tx(full(s), STAGE_BYTES);
          tma2d(st, &map_x, full(s), k * BK, m_i * BM);
          // N-atoms: gate [128 n, +64), [+64, +128), up [I + 128 n, ...)
#pragma unroll
          for (int i = 0; i < 4; ++i)
            tma2d(st + A_BYTES + i * 8192, &map_w, full(s),
                  (i < 2 ? 0 : I) + n_i * 128 + (i & 1) * 64, k * BK);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      // kind::f16, bf16 A/B, f32 D, A K-major, B MN-major, N = 256, M = 128
      constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                                 ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      int s = 0, it = 0;
      uint32_t ph = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
        const int b = it & 1;
        mbar_wait(aempty(b), (uint32_t)(((it >> 1) & 1) ^ 1));
        fence_after();
        const uint32_t acc = tmem + (uint32_t)(b * 256);
        for (int k = 0; k < kt; ++k) {
          mbar_wait(full(s), ph);
          fence_after();
          const uint32_t st = base + s * STAGE_BYTES;
          const uint64_t ad = sdesc(st, 16, 1024), bd = sdesc(st + A_BYTES, 8192, 1024);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk)
            mma(acc, ad + (uint64_t)((kk * 32) >> 4), bd + (uint64_t)((kk * 2048) >> 4), IDESC,
                (k | kk) ? 1u : 0u);
          commit(empty(s));
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        commit(afull(b));
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3, row = q * 32 + lane;  // TMEM lane quarter = warp % 4
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    int it = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x, ++it) {
      const int b = it & 1;
      int m_i, n_i;
      tm.at(t, m_i, n_i);
      mbar_wait(afull(b), (uint32_t)((it >> 1) & 1));
      __syncwarp();
      fence_after();
      const uint32_t acc = tmem + (uint32_t)(b * 256) + lane_off;
      const int64_t grow = (int64_t)m_i * BM + row;
      const bool valid = grow < M;
      uint4* dst = reinterpret_cast<uint4*>(act + grow * ld_act + (int64_t)n_i * 128);
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t g[32], u[32];
        ld32(acc + c * 32, g);
        ld32(acc + 128 + c * 32, u);
        ld_wait(g);  // waits for both loads
        ld_wait(u);
        if (valid) {
          float a[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const float x = __uint_as_float(g[e]);
            a[e] = x / (1.f + __expf(-x)) * __uint_as_float(u[e]);
          }
#pragma unroll
          for (int e = 0; e < 4; ++e)
            dst[c * 4 + e] = make_uint4(pack(a[8 * e], a[8 * e + 1]), pack(a[8 * e + 2], a[8 * e + 3]),
                                        pack(a[8 * e + 4], a[8 * e + 5]),
                                        pack(a[8 * e + 6], a[8 * e + 7]));
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

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return (PFN_cuTensorMapEncodeTiled_v12000)p;
  }();
  return fn;
}
// 2-D bf16 map: `inner` contiguous elements per row, `outer` rows of
// `ld` elements, box b0 x b1, SWIZZLE_128B
static int map2d(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                 uint32_t b0, uint32_t b1) {
  auto enc = encode_fn();
  if (!enc) return fail(CT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {b0, b1};
  cuuint32_t es[2] = {1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CT_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return CT_OK;
}

static int sm_count() {
  static const int n = [] {
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
      cudaGetLastError();
      return 148;
    }
    return v;
  }();
  return n;
}

}  // namespace gm
}  // namespace ct

using namespace ct;

extern "C" int ct_gemm_swiglu(const void* x, int64_t M, int64_t K, int64_t ldx, const void* w,
                              int64_t I, int64_t ldw, void* act, int64_t ld_act, void* stream) {
  if (M < 1 || K < 1 || I < 1)
    return fail(CT_ERR_SHAPE, "gemm_swiglu geometry M=%lld K=%lld I=%lld", (long long)M,
                (long long)K, (long long)I);
  if (K % gm::BK || I % 128 || ldx < K || ldw < 2 * I || ld_act < I)
    return fail(CT_ERR_UNSUPPORTED, "gemm_swiglu needs K %% 64 == 0, I %% 128 == 0 (K=%lld I=%lld)",
                (long long)K, (long long)I);
  if (!x || !w || !act) return fail(CT_ERR_PARAM, "null tensor");
  if ((((uintptr_t)x | (uintptr_t)w | (uintptr_t)act) & 15) || ldx % 8 || ldw % 8 || ld_act % 8)
    return fail(CT_ERR_UNSUPPORTED, "gemm_swiglu needs 16-byte aligned rows");
  if (M > INT32_MAX / 2) return fail(CT_ERR_UNSUPPORTED, "M too large");
  CUtensorMap mx, mw;
  int rc;
  if ((rc = gm::map2d(&mx, x, (uint64_t)K, (uint64_t)M, (uint64_t)ldx, 64, gm::BM))) return rc;
  if ((rc = gm::map2d(&mw, w, (uint64_t)(2 * I), (uint64_t)K, (uint64_t)ldw, 64, 64))) return rc;
  CT_CUDA(cudaFuncSetAttribute(gm::gemm_swiglu_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)gm::SMEM));
  const int64_t tiles = ((M + gm::BM - 1) / gm::BM) * (I / 128);
  const unsigned grid = (unsigned)std::min<int64_t>(tiles, gm::sm_count());
  // M-tiles per band: an A slice of at most ~60 MB (L2 is 126 MB over two
  // dies; a single 81 MB band measured 4 % slower than two), bands of
  // equal size
  const int64_t mt = (M + gm::BM - 1) / gm::BM;
  const int64_t fit = std::max<int64_t>(1, (int64_t)60e6 / (gm::BM * K * 2));
  const int64_t nbands = (mt + fit - 1) / fit;
  const int band_m = (int)((mt + nbands - 1) / nbands);
  gm::gemm_swiglu_kernel<<<grid, 192, gm::SMEM, (cudaStream_t)stream>>>(
      mx, mw, (__nv_bfloat16*)act, (int)M, (int)I, (int)K, ld_act, band_m);
  return check_launch("gemm_swiglu_kernel");
}
