// Gate/up projection with the SwiGLU activation fused into the epilogue, on
// the 5th-gen tensor cores (sm_100a).  Replaces, for the bf16 step, the pair
//     gu = x @ W_gu (cuBLAS)   ->   act = silu(gu[:, :I]) * gu[:, I:]  (ct_mlp_act)
// of ct/toymodel.py:186 (the MLP, as SwiGLU in the restated Llama/Mistral
// geometry): the [M, 2I] gate/up product never reaches HBM, and the
// activation is computed from the f32 accumulators.
//
// Default: a CTA pair (cluster of 2 on one TPC, tcgen05 cta_group::2).  One
// MMA tile = 256 rows x 256 accumulator columns = 128 gate + the matching 128
// up columns, so one N-tile yields 128 finished activation columns; CTA r of
// the pair holds rows [128 r, 128 r + 128) of x and half of B (r = 0 the gate
// columns, r = 1 the up columns), and its TMEM receives all 256 columns of
// its own 128 rows.  Per CTA and 64-deep K stage: 16 KiB of A + 16 KiB of B
// (the 1-SM M128 N256 form reads 48 KiB of operands from shared memory for
// the same 128 x 256 x 64 MACs per SM).  Config-2 shape (4992 x 4096 x
// 2 x 14336) under ncu: 743.5 us at 1.435 GHz = 1.58 PFLOP/s, 96 % of the
// dense bf16 peak at that clock (profiles/round2_gemm_swiglu_ncu.md).
//   warp 0   TMA producer (both CTAs): A box 64 K x 128 rows (K-major), two
//            B boxes 64 N x 64 K (MN-major), SWIZZLE_128B; completion bytes
//            of both CTAs land on the leader's full barrier
//   warp 1   TMEM allocation (both CTAs); MMA issuer (leader only):
//            tcgen05.mma.cta_group::2 kind::f16 M256 N256 K16, commits
//            multicast to the stage / accumulator barriers of both CTAs
//   warps 2-5 epilogue (both CTAs): one TMEM lane (= output row) per thread,
//            silu(g) * u in f32, bf16 16-byte stores; each warp releases the
//            accumulator on the leader's barrier
// The same kernel serves the step's other projections through ct_gemm_bf16
// (epilogue STORE: bf16 out = x @ w; ADD: f32 out += x @ w), with tiles of
// 256 x 256 output columns (128 per CTA of B) or 256 x 128 when N % 256 != 0.
// NCTA = 1 (CT_GEMM_1SM=1) is the single-SM form (M128 N256, all four B
// boxes in one CTA), kept for A/B.
// TMEM holds two 256-column accumulators, so the epilogue of tile t runs
// under the MMAs of tile t+1.  Persistent: one CTA (pair) per SM (TPC) walks
// the tiles N-major within L2-sized bands of M-tiles (TileMap), so
// consecutive pairs share the B tile and the A slice stays in L2.  Rows past
// M are zero-filled by TMA and not stored.
#include "common.cuh"

#include <cuda.h>
#include <algorithm>
#include <cudaTypedefs.h>

namespace ct {
namespace gm {

constexpr int BM = 128, BK = 64;  // rows per CTA, K per stage
constexpr int A_BYTES = BM * BK * 2;          // 16 KiB
template <int NCTA, int BNT>  // BNT: accumulator columns per tile (256 or 128)
struct Cfg {
  static constexpr int ATOMS = BNT / 64 / NCTA;  // 64 x 64 B atoms held by this CTA
  static constexpr int B_BYTES = ATOMS * 8192;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (192 * 1024) / STAGE_BYTES > 8 ? 8 : (192 * 1024) / STAGE_BYTES;
  static constexpr int NBAR = 2 * STAGES + 4;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + NBAR * 8 + 16 + 1024;
};
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
// try_wait suspend-time hint (ns): waiting threads (4 epilogue warps, the
// producer and the MMA thread per CTA) may sleep instead of re-issuing the
// poll.  In-step A/B (tools/gemm_power_ab.sh, profiles/round2_gemm_power_ab.txt):
// -0.3 to -0.5 ms per request at configs 2 and 3 under the power cap.
// -DCT_GEMM_SUSPEND_NS=0 builds the plain spin.
#ifndef CT_GEMM_SUSPEND_NS
#define CT_GEMM_SUSPEND_NS 1000000
#endif
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t par) {
#if CT_GEMM_SUSPEND_NS
  // waiting threads may be suspended up to the hint instead of re-issuing
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLW:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra LD;\n\tbra LW;\n\tLD:\n\t}" ::"r"(b),
      "r"(par), "n"(CT_GEMM_SUSPEND_NS)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLW:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra LD;\n\tbra LW;\n\tLD:\n\t}" ::"r"(b),
      "r"(par)
      : "memory");
#endif
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
// ---- CTA-pair (cta_group::2) forms
// TMA into this CTA's shared memory, completion bytes on the leader's barrier
// (clearing the peer bit of the shared::cluster address selects CTA 0)
__device__ __forceinline__ void tma2d_pair(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0,
                                           int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(m), "r"(bar & 0xFEFFFFFFu), "r"(c0), "r"(c1)
      : "memory");
}
// arrive on the same barrier of both CTAs when the issued MMAs complete
__device__ __forceinline__ void commit_pair(uint32_t b) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(b),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mma_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t id,
                                         uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
// arrive on barrier `b` (a local shared address) of cluster CTA 0
__device__ __forceinline__ void mbar_arrive_leader(uint32_t b) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, 0;\n\t"
      "mbarrier.arrive.release.cluster.shared::cluster.b64 _, [ra];\n\t}" ::"r"(b)
      : "memory");
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
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

// epilogues: SWIGLU act = silu(g) * u (bf16, B columns = gate | up halves of
// width I); STORE out = x @ w (bf16); ADD out += x @ w (f32 residual, the
// beta = 1 GEMM of the O- and down-projections)
// QKV: the q|k|v projection with the K4 epilogue of ct_qkv_rope_scatter
// fused (bf16, head_dim 128, adjacent RoPE pairs): q heads rotated at the
// row's position -> q_out [M, Hq, 128]; k heads rotated -> k cache row pos;
// v heads -> v cache row pos.  RoPE runs on the f32 accumulators.
enum Mode { SWIGLU = 0, STORE = 1, ADD = 2, QKV = 3 };

struct QkvEpi {
  const int32_t* pos;     // [M] global positions of the rows
  const float4* table;    // [n_ctx][64] (cos, sin) f32 pairs, read as float4
  __nv_bfloat16* q;       // [M][hq][128]
  __nv_bfloat16* kc;      // cache rows [n_ctx] x crs
  __nv_bfloat16* vc;
  int64_t crs;
  int hq, hkv;
};

template <int NCTA, int MODE, int BNT>
__global__ void __launch_bounds__(192, 1)
gemm_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w,
            void* __restrict__ out, int M, int N, int K, int64_t ld_out, int band_m,
            const QkvEpi qe) {
  // N: activation width I (SWIGLU) or output columns
  static_assert(MODE != SWIGLU || BNT == 256, "SWIGLU tiles pair 128 gate + 128 up columns");
  using C = Cfg<NCTA, BNT>;
  constexpr int STAGES = C::STAGES, STAGE_BYTES = C::STAGE_BYTES;
  constexpr bool PAIR = NCTA == 2;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;  // the same offset in both CTAs of a pair
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t bar = base + STAGES * STAGE_BYTES;
  auto full = [&](int s) { return bar + s * 8; };
  auto empty = [&](int s) { return bar + (STAGES + s) * 8; };
  auto afull = [&](int b) { return bar + (2 * STAGES + b) * 8; };
  auto aempty = [&](int b) { return bar + (2 * STAGES + 2 + b) * 8; };
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int rank = PAIR ? (int)cluster_rank() : 0;
  // TMEM address slot at the same offset in both CTAs: the pair allocation
  // writes it for the pair (a per-rank slot leaves rank 1's unwritten), so
  // racecheck reports the two CTAs' allocations writing the same value here
  // (profiles/round2_sanitizer.md); both complete before the cluster barrier
  // that precedes the read
  uint32_t* tptr = reinterpret_cast<uint32_t*>(gbase + STAGES * STAGE_BYTES + C::NBAR * 8);
  const int unit = blockIdx.x / NCTA, units = gridDim.x / NCTA;  // pair index / pairs
  constexpr int TM = BM * NCTA;                                   // rows per MMA tile
  const int mt = (M + TM - 1) / TM, nt = MODE == SWIGLU ? N / 128 : N / BNT;
  const int tiles = mt * nt, kt = K / BK;
  const TileMap tm{mt, nt, band_m};
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full(s), 1);  // the leader's expect_tx (pair: both CTAs' bytes)
      mbar_init(empty(s), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(afull(b), 1);
      mbar_init(aempty(b), 4 * NCTA);  // one arrival per epilogue warp of the pair
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       su32(tptr)), "n"(2 * BNT)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       su32(tptr)), "n"(2 * BNT)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  fence_before();
  if constexpr (PAIR)
    cluster_sync();  // barrier inits and the allocation visible to the peer
  else
    __syncthreads();
  fence_after();
  const uint32_t tmem = *tptr;
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int t = unit; t < tiles; t += units) {
        int m_i, n_i;
        tm.at(t, m_i, n_i);
        const int row0 = m_i * TM + rank * BM;
        for (int k = 0; k < kt; ++k) {
          mbar_wait(empty(s), ph ^ 1);
          const uint32_t st = base + s * STAGE_BYTES;
          if constexpr (PAIR) {
            if (rank == 0) mbar_expect_tx(full(s), 2 * STAGE_BYTES);
            tma2d_pair(st, &map_x, full(s), k * BK, row0);
            // this CTA's half of B: SWIGLU rank 0 gate [128 n, +128), rank 1 up
            // [N + 128 n, ...); otherwise columns [256 n + 128 rank, +128)
            const int c0 = MODE == SWIGLU ? rank * N + n_i * 128 : n_i * BNT + rank * (BNT / 2);
#pragma unroll
            for (int i = 0; i < C::ATOMS; ++i)
              tma2d_pair(st + A_BYTES + i * 8192, &map_w, full(s), c0 + i * 64, k * BK);
          } else {
            mbar_expect_tx(full(s), STAGE_BYTES);
            tma2d(st, &map_x, full(s), k * BK, row0);
            // N-atoms: SWIGLU gate [128 n, +64), [+64, +128), up [N + 128 n, ...);
            // otherwise [BNT n + 64 i, +64)
#pragma unroll
            for (int i = 0; i < C::ATOMS; ++i)
              tma2d(st + A_BYTES + i * 8192, &map_w, full(s),
                    MODE == SWIGLU ? (i < 2 ? 0 : N) + n_i * 128 + (i & 1) * 64
                                   : n_i * BNT + i * 64,
                    k * BK);
          }
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && rank == 0) {
      // kind::f16, bf16 A/B, f32 D, A K-major, B MN-major, N = BNT, M = 128 NCTA
      constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) |
                                 ((uint32_t)(BNT >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
      int s = 0, it = 0;
      uint32_t ph = 0;
      for (int t = unit; t < tiles; t += units, ++it) {
        const int b = it & 1;
        mbar_wait(aempty(b), (uint32_t)(((it >> 1) & 1) ^ 1));
        fence_after();
        const uint32_t acc = tmem + (uint32_t)(b * BNT);
        for (int k = 0; k < kt; ++k) {
          mbar_wait(full(s), ph);
          fence_after();
          const uint32_t st = base + s * STAGE_BYTES;
          const uint64_t ad = sdesc(st, 16, 1024), bd = sdesc(st + A_BYTES, 8192, 1024);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t a = ad + (uint64_t)((kk * 32) >> 4), bb = bd + (uint64_t)((kk * 2048) >> 4);
            if constexpr (PAIR)
              mma_pair(acc, a, bb, IDESC, (k | kk) ? 1u : 0u);
            else
              mma(acc, a, bb, IDESC, (k | kk) ? 1u : 0u);
          }
          if constexpr (PAIR)
            commit_pair(empty(s));
          else
            commit(empty(s));
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        if constexpr (PAIR)
          commit_pair(afull(b));
        else
          commit(afull(b));
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int q = warp & 3, row = q * 32 + lane;  // TMEM lane quarter = warp % 4
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    int it = 0;
    for (int t = unit; t < tiles; t += units, ++it) {
      const int b = it & 1;
      int m_i, n_i;
      tm.at(t, m_i, n_i);
      mbar_wait(afull(b), (uint32_t)((it >> 1) & 1));
      __syncwarp();
      fence_after();
      const uint32_t acc = tmem + (uint32_t)(b * BNT) + lane_off;
      const int64_t grow = (int64_t)m_i * TM + rank * BM + row;
      const bool valid = grow < M;
      if constexpr (MODE == SWIGLU) {
        uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(out) + grow * ld_out +
                                              (int64_t)n_i * 128);
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
              dst[c * 4 + e] =
                  make_uint4(pack(a[8 * e], a[8 * e + 1]), pack(a[8 * e + 2], a[8 * e + 3]),
                             pack(a[8 * e + 4], a[8 * e + 5]), pack(a[8 * e + 6], a[8 * e + 7]));
          }
        }
      } else if constexpr (MODE == STORE) {
        uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(out) + grow * ld_out +
                                              (int64_t)n_i * BNT);
#pragma unroll 1
        for (int c = 0; c < BNT / 32; ++c) {
          uint32_t v[32];
          ld32(acc + c * 32, v);
          ld_wait(v);
          if (valid) {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              dst[c * 4 + e] = make_uint4(
                  pack(__uint_as_float(v[8 * e]), __uint_as_float(v[8 * e + 1])),
                  pack(__uint_as_float(v[8 * e + 2]), __uint_as_float(v[8 * e + 3])),
                  pack(__uint_as_float(v[8 * e + 4]), __uint_as_float(v[8 * e + 5])),
                  pack(__uint_as_float(v[8 * e + 6]), __uint_as_float(v[8 * e + 7])));
          }
        }
      } else if constexpr (MODE == QKV) {
        const int64_t pos = valid ? (int64_t)__ldg(qe.pos + grow) : 0;
#pragma unroll 1
        for (int c = 0; c < BNT / 32; ++c) {
          uint32_t v[32];
          ld32(acc + c * 32, v);
          ld_wait(v);
          if (valid) {
            const int col = n_i * BNT + c * 32;
            const int head = col >> 7, d0 = col & 127;
            uint4* dst;
            uint32_t pk[16];
            if (head < qe.hq + qe.hkv) {
              dst = reinterpret_cast<uint4*>(
                  head < qe.hq ? qe.q + grow * (int64_t)qe.hq * 128 + col
                               : qe.kc + pos * qe.crs + (head - qe.hq) * 128 + d0);
              // 16 adjacent pairs (2j, 2j+1), j = d0/2 + e: 8 float4 of (cos, sin)
              const float4* t = qe.table + pos * 32 + d0 / 4;
#pragma unroll
              for (int e = 0; e < 8; ++e) {
                const float4 cs = __ldg(t + e);
                const float x0 = __uint_as_float(v[4 * e]), y0 = __uint_as_float(v[4 * e + 1]);
                const float x1 = __uint_as_float(v[4 * e + 2]), y1 = __uint_as_float(v[4 * e + 3]);
                pk[2 * e] = pack(x0 * cs.x - y0 * cs.y, x0 * cs.y + y0 * cs.x);
                pk[2 * e + 1] = pack(x1 * cs.z - y1 * cs.w, x1 * cs.w + y1 * cs.z);
              }
            } else {
              dst = reinterpret_cast<uint4*>(qe.vc + pos * qe.crs +
                                             (head - qe.hq - qe.hkv) * 128 + d0);
#pragma unroll
              for (int e = 0; e < 16; ++e)
                pk[e] = pack(__uint_as_float(v[2 * e]), __uint_as_float(v[2 * e + 1]));
            }
#pragma unroll
            for (int e = 0; e < 4; ++e)
              dst[e] = make_uint4(pk[4 * e], pk[4 * e + 1], pk[4 * e + 2], pk[4 * e + 3]);
          }
        }
      } else {
        float4* dst = reinterpret_cast<float4*>(static_cast<float*>(out) + grow * ld_out +
                                                (int64_t)n_i * BNT);
#pragma unroll 1
        for (int c = 0; c < BNT / 32; ++c) {
          uint32_t v[32];
          ld32(acc + c * 32, v);
          float4 h[8];
          if (valid) {
#pragma unroll
            for (int e = 0; e < 8; ++e) h[e] = dst[c * 8 + e];
          }
          ld_wait(v);
          if (valid) {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              dst[c * 8 + e] = make_float4(h[e].x + __uint_as_float(v[4 * e]),
                                           h[e].y + __uint_as_float(v[4 * e + 1]),
                                           h[e].z + __uint_as_float(v[4 * e + 2]),
                                           h[e].w + __uint_as_float(v[4 * e + 3]));
          }
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (PAIR)
          mbar_arrive_leader(aempty(b));
        else
          mbar_arrive(aempty(b));
      }
    }
  }
  fence_before();
  if constexpr (PAIR)
    cluster_sync();  // both CTAs done with TMEM and with each other's barriers
  else
    __syncthreads();
  if (warp == 1) {
    fence_after();
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * BNT)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(2 * BNT)
                   : "memory");
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

namespace {

template <int MODE, int BNT>
int launch_mode(int ncta, const CUtensorMap& mx, const CUtensorMap& mw, void* out, int M, int N,
                int K, int64_t ld_out, int band_m, int units, cudaStream_t stream,
                const gm::QkvEpi& qe) {
  cudaLaunchConfig_t lc = {};
  cudaLaunchAttribute at[1];
  lc.gridDim = dim3((unsigned)(units * ncta));
  lc.blockDim = dim3(192);
  lc.stream = stream;
  if (ncta == 2) {
    CT_CUDA(cudaFuncSetAttribute(gm::gemm_kernel<2, MODE, BNT>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)gm::Cfg<2, BNT>::SMEM));
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    lc.dynamicSmemBytes = gm::Cfg<2, BNT>::SMEM;
    CT_CUDA(cudaLaunchKernelEx(&lc, gm::gemm_kernel<2, MODE, BNT>, mx, mw, out, M, N, K, ld_out,
                               band_m, qe));
  } else {
    CT_CUDA(cudaFuncSetAttribute(gm::gemm_kernel<1, MODE, BNT>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)gm::Cfg<1, BNT>::SMEM));
    lc.dynamicSmemBytes = gm::Cfg<1, BNT>::SMEM;
    CT_CUDA(cudaLaunchKernelEx(&lc, gm::gemm_kernel<1, MODE, BNT>, mx, mw, out, M, N, K, ld_out,
                               band_m, qe));
  }
  return check_launch(MODE == gm::SWIGLU ? "gemm_swiglu_kernel"
                      : MODE == gm::QKV  ? "gemm_qkv_rope_kernel"
                                         : "gemm_bf16_kernel");
}

// x [M][K] bf16 (row stride ldx) times w [K][wcols] bf16 (row stride ldw);
// N = activation width (SWIGLU, wcols = 2N) or output columns (wcols = N)
int launch(int mode, const void* x, int64_t M, int64_t K, int64_t ldx, const void* w,
           int64_t wcols, int64_t ldw, int64_t N, void* out, int64_t ld_out, int out_bytes,
           void* stream, const gm::QkvEpi& qe = gm::QkvEpi{}) {
  if (M < 1 || K < 1 || N < 1)
    return fail(CT_ERR_SHAPE, "gemm geometry M=%lld K=%lld N=%lld", (long long)M, (long long)K,
                (long long)N);
  if (K % gm::BK || N % 128 || ldx < K || ldw < wcols || ld_out < N)
    return fail(CT_ERR_UNSUPPORTED, "gemm needs K %% 64 == 0 and N %% 128 == 0 (K=%lld N=%lld)",
                (long long)K, (long long)N);
  if (!x || !w || !out) return fail(CT_ERR_PARAM, "null tensor");
  if ((((uintptr_t)x | (uintptr_t)w | (uintptr_t)out) & 15) || ldx % 8 || ldw % 8 ||
      (ld_out * out_bytes) % 16)
    return fail(CT_ERR_UNSUPPORTED, "gemm needs 16-byte aligned rows");
  if (M > INT32_MAX / 2 || N > INT32_MAX / 4) return fail(CT_ERR_UNSUPPORTED, "gemm too large");
  CUtensorMap mx, mw;
  int rc;
  if ((rc = gm::map2d(&mx, x, (uint64_t)K, (uint64_t)M, (uint64_t)ldx, 64, gm::BM))) return rc;
  if ((rc = gm::map2d(&mw, w, (uint64_t)wcols, (uint64_t)K, (uint64_t)ldw, 64, 64))) return rc;
  // CT_GEMM_1SM=1 (read once): the single-SM form, for A/B
  static const bool one_sm = [] {
    const char* e = getenv("CT_GEMM_1SM");
    return e && e[0] == '1';
  }();
  const int ncta = one_sm ? 1 : 2;
  const int64_t tm_rows = (int64_t)gm::BM * ncta;
  const int64_t mt = (M + tm_rows - 1) / tm_rows, slots = gm::sm_count() / ncta;
  // tile width (accumulator columns): 256 (SWIGLU: 128 gate + 128 up).
  // 128-wide tiles only when N % 256 != 0: at N = 128 each MMA still reads
  // the whole A operand from shared memory for half the MACs, and measured
  // 25-33 % slower than 256-wide tiles on the step's projections even where
  // they fill the last wave better (tools/gemm_proj_bench.py)
  const bool narrow = mode != gm::SWIGLU && mode != gm::QKV && N % 256;
  const int64_t tiles = mt * (mode == gm::SWIGLU ? N / 128 : N / (narrow ? 128 : 256));
  // M-tiles per band: an A slice of at most ~60 MB (L2 is 126 MB over two
  // dies), bands of equal size.  Standalone (tools/gemm_band_sweep.sh) 40
  // and 60 MB tie at 2K / 5K / 10K rows and 40 MB wins at 32K rows (one band
  // -26 %); inside the power-capped step 60 MB measured 0.4-0.5 ms faster
  // per request at configs 2 and 3 (config 2's 41 MB x stays one band, so W
  // is read from HBM once instead of twice), and the step's fused calls stay
  // below 16K rows
  static const int64_t band_bytes = [] {  // CT_GEMM_BAND_MB (read once): sweep switch
    const char* e = getenv("CT_GEMM_BAND_MB");
    return (int64_t)((e && atoi(e) > 0) ? atoi(e) : 60) * 1000000;
  }();
  const int64_t fit = std::max<int64_t>(1, band_bytes / (tm_rows * K * 2));
  const int64_t nbands = (mt + fit - 1) / fit;
  const int band_m = (int)((mt + nbands - 1) / nbands);
  const int units = (int)std::min<int64_t>(tiles, slots);
  const cudaStream_t st = (cudaStream_t)stream;
  const int m = (int)M, n = (int)N, k = (int)K;
  if (mode == gm::SWIGLU)
    return launch_mode<gm::SWIGLU, 256>(ncta, mx, mw, out, m, n, k, ld_out, band_m, units, st, qe);
  if (mode == gm::QKV)
    return launch_mode<gm::QKV, 256>(ncta, mx, mw, out, m, n, k, ld_out, band_m, units, st, qe);
  if (mode == gm::STORE)
    return narrow ? launch_mode<gm::STORE, 128>(ncta, mx, mw, out, m, n, k, ld_out, band_m, units, st, qe)
                  : launch_mode<gm::STORE, 256>(ncta, mx, mw, out, m, n, k, ld_out, band_m, units, st, qe);
  return narrow ? launch_mode<gm::ADD, 128>(ncta, mx, mw, out, m, n, k, ld_out, band_m, units, st, qe)
                : launch_mode<gm::ADD, 256>(ncta, mx, mw, out, m, n, k, ld_out, band_m, units, st, qe);
}

}  // namespace

extern "C" int ct_gemm_swiglu(const void* x, int64_t M, int64_t K, int64_t ldx, const void* w,
                              int64_t I, int64_t ldw, void* act, int64_t ld_act, void* stream) {
  return launch(gm::SWIGLU, x, M, K, ldx, w, 2 * I, ldw, I, act, ld_act, 2, stream);
}

extern "C" int ct_gemm_bf16(const void* x, int64_t M, int64_t K, int64_t ldx, const void* w,
                            int64_t N, int64_t ldw, void* out, int64_t ld_out, int out_dtype,
                            int accumulate, void* stream) {
  if (out_dtype == CT_BF16 && !accumulate)
    return launch(gm::STORE, x, M, K, ldx, w, N, ldw, N, out, ld_out, 2, stream);
  if (out_dtype == CT_F32 && accumulate)
    return launch(gm::ADD, x, M, K, ldx, w, N, ldw, N, out, ld_out, 4, stream);
  return fail(CT_ERR_UNSUPPORTED, "gemm_bf16: bf16 store or f32 accumulate only");
}

// q|k|v projection + RoPE + cache scatter in one kernel (bf16, head_dim 128,
// adjacent pairing): replaces torch.mm(x, wqkv) -> ct_qkv_rope_scatter.
extern "C" int ct_gemm_qkv_rope(const void* x, int64_t M, int64_t K, int64_t ldx, const void* w,
                                int64_t ldw, const int32_t* positions, const void* table,
                                int64_t Hq, int64_t Hkv, int64_t D, void* q_out, void* k_cache,
                                void* v_cache, int64_t cache_row_stride, void* stream) {
  if (D != 128) return fail(CT_ERR_UNSUPPORTED, "gemm_qkv_rope: head_dim %lld != 128", (long long)D);
  if (Hq < 1 || Hkv < 1 || Hq % Hkv)
    return fail(CT_ERR_SHAPE, "gemm_qkv_rope: Hq=%lld Hkv=%lld", (long long)Hq, (long long)Hkv);
  if (!positions || !table || !q_out || !k_cache || !v_cache) return fail(CT_ERR_PARAM, "null tensor");
  if ((((uintptr_t)table | (uintptr_t)q_out | (uintptr_t)k_cache | (uintptr_t)v_cache) & 15) ||
      cache_row_stride % 8 || cache_row_stride < Hkv * D)
    return fail(CT_ERR_UNSUPPORTED, "gemm_qkv_rope needs 16-byte aligned rows");
  const int64_t N = (Hq + 2 * Hkv) * D;
  if (N % 256) return fail(CT_ERR_UNSUPPORTED, "gemm_qkv_rope: (Hq + 2 Hkv) must be even");
  if (M == 0) return CT_OK;
  gm::QkvEpi qe{positions, static_cast<const float4*>(table), static_cast<__nv_bfloat16*>(q_out),
                static_cast<__nv_bfloat16*>(k_cache), static_cast<__nv_bfloat16*>(v_cache),
                cache_row_stride, (int)Hq, (int)Hkv};
  return launch(gm::QKV, x, M, K, ldx, w, N, ldw, N, q_out, N, 2, stream, qe);
}
