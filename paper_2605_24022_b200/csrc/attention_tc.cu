// (4) Selective-recompute attention on the 5th-gen tensor cores (sm_100a):
// tcgen05.mma with fp32 accumulators in TMEM, bf16 operands staged by TMA.
// Replaces the attention of ct/toymodel.py:176-183 (q = selected rows + suffix
// at global positions, keys/values = the full blended cache, key j visible to
// a query iff j <= its position).
//
// Tile = 128 TMEM lanes = (128/G queries) x (G q-heads of one kv-head), so a
// K/V tile staged once serves the whole GQA group.  Per 128-key block:
//   S = Q K^T      tcgen05.mma  M128 N128 K16 x8, A = Q smem, B = K smem -> TMEM
//   softmax        one thread per row: tcgen05.ld S row, mask by position,
//                  exp2 against a lazily rescaled running max, P (bf16) back
//                  into TMEM over S
//   O += P V       tcgen05.mma  M128 N128 K16 x8, A = P TMEM, B = V smem (MN-major)
// Warp roles: warps 0-7 softmax/epilogue (4 per tile of a ping-pong pair),
// warp 8 TMA producer (5-slot K/V ring + Q), warp 9 MMA issuer (+ TMEM alloc).
// Timing-probe and CTA-pair variants measured in round 1 are not built into
// the product library (profiles/round1_attention_variants.md; git history).
#include "common.cuh"

#include <cuda.h>
#include <algorithm>
#include <type_traits>
#include <cudaTypedefs.h>

namespace ct {

namespace tc {

// Diagnostic timeline (tools/build_trace.sh builds a separate library with
// CT_ATT_TRACE): SM clock at softmax start / end and MMA PV / S issue of the
// first unit of CTA 0, per tile and block.  Compiled out of the product.
#ifdef CT_ATT_TRACE
__device__ unsigned long long g_trace[14][2][512];
#define CT_TRACE(ev_, t_, j_, cond_) \
  if ((cond_) && blockIdx.x == 0 && (j_) < 512) g_trace[ev_][t_][j_] = clock64();
#else
#define CT_TRACE(ev_, t_, j_, cond_)
#endif

constexpr int TILE_M = 128;   // TMEM lanes / MMA M
constexpr int BLK_N = 128;    // keys per block
constexpr int HD = 128;       // head dim
constexpr int KV_SLOTS = 5;
constexpr int ATOM_BYTES = 128 * 64 * 2;      // [128 rows][64 bf16] swizzle-128B half tile
constexpr int TILE_BYTES = 2 * ATOM_BYTES;    // 32 KiB: 128 rows x 128 bf16
constexpr float LAZY_THRESH = 8.0f;           // log2 units


__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// try_wait with a suspend-time hint (ns): waiting warps may sleep instead of
// re-issuing the poll, as gemm.cu's CT_GEMM_SUSPEND_NS.  A/B vs the plain spin
// (tools/att_suspend_ab.sh, profiles/round2_attention_suspend_ab.txt): outputs
// bit-identical, in-step launch -0.3 % (config 2) / -0.7 % (config 3), p50
// -0.1 / -0.8 ms per request, every rep; a 2 us hint is neutral to slower.
// -DCT_TC_SUSPEND_NS=0 builds the plain spin.
#ifndef CT_TC_SUSPEND_NS
#define CT_TC_SUSPEND_NS 1000000
#endif
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
#if CT_TC_SUSPEND_NS
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t}" ::"r"(bar),
      "r"(parity), "n"(CT_TC_SUSPEND_NS)
      : "memory");
  return;
#endif
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\t"
      "bra LAB_WAIT;\n\t"
      "DONE:\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
      : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}

// A operand from TMEM (.kind::f16, A K-major packed bf16x2 along columns).
__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accum)
      : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}

// 32 consecutive TMEM columns of this thread's lane.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// wait::ld, threading the registers through so uses cannot move above it
__device__ __forceinline__ void tmem_wait_ld32(uint32_t* r) {
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
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]),
      "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]),
      "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// Shared-memory matrix descriptor, SWIZZLE_128B (sm100 version bit set).
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;          // descriptor version (Blackwell)
  d |= (uint64_t)2 << 61;          // SWIZZLE_128B
  return d;
}

// Instruction descriptor: kind::f16, bf16 A/B, f32 D, M = 128*CTAS, N=128.
__host__ __device__ constexpr uint32_t idesc_bf16(bool b_mn_major, int m = TILE_M) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) |
         ((uint32_t)(BLK_N >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// --- packed fp32 (FFMA2 / FADD2) and 3-input max helpers (sm_100a) ----------
__device__ __forceinline__ uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk2(uint64_t v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float max3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// 2^x for x <= ~8 on the FMA pipe: round-to-nearest split x = n + f, f in
// [-1/2, 1/2], degree-3 minimax 2^f (max rel err 7.5e-5, below bf16 P
// rounding), exponent add.  x clamped at -126 (result ~1e-38, i.e. zero).
__device__ __forceinline__ void exp2_poly2(uint64_t x2, uint32_t& o0, uint32_t& o1) {
  float a, b;
  upk2(x2, a, b);
  const uint64_t xc = pk2(fmaxf(a, -126.f), fmaxf(b, -126.f));
  const uint64_t t = fadd2(xc, pk2(12582912.f, 12582912.f));
  const uint64_t rr = fadd2(t, pk2(-12582912.f, -12582912.f));
  const uint64_t f = ffma2(rr, pk2(-1.f, -1.f), xc);
  uint64_t pp = ffma2(f, pk2(0.05517025291919708f, 0.05517025291919708f),
                      pk2(0.24260790646076202f, 0.24260790646076202f));
  pp = ffma2(pp, f, pk2(0.693260908126831f, 0.693260908126831f));
  pp = ffma2(pp, f, pk2(0.9999282956123352f, 0.9999282956123352f));
  o0 = (uint32_t)pp + ((uint32_t)t << 23);
  o1 = (uint32_t)(pp >> 32) + ((uint32_t)(t >> 32) << 23);
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

struct Params {
  const int32_t* qpos;
  __nv_bfloat16* out;
  float* out_f32;
  int A, Hq, Hkv, G, QB;  // G = Hq/Hkv rows per query, QB = 128/G queries per tile
  int n_ctx;
  int n_qblocks;
  float scale_log2;
  float lazy_thresh;
};


// ---------------------------------------------------------------------------
// Persistent ping-pong kernel.  A work unit is two adjacent 128-row query
// tiles (X = 0, 1) of one kv head; they share every K/V tile.  One CTA per SM
// walks its units (longest first, snake order over the CTAs) with ONE TMEM
// allocation and one barrier set for its lifetime; the TMA producer runs into
// the next unit's Q and K/V while the softmax warps finish the current
// unit's epilogue.  TMEM = S_0 | S_1 | O_0 | O_1 (128 columns each; P_X, bf16,
// overwrites the first half of S_X and is the A operand of the PV MMA).  One
// softmax thread per tile row (warps 0-3 tile 0, warps 4-7 tile 1: every SMSP
// runs one warp of each tile), MMA order
//     S_0(0) S_1(0) | PV_0(j) S_0(j+1) PV_1(j) S_1(j+1) | ...
// (S_X(j+1) overwrites P_X(j): it is issued right behind PV_X(j), the
// tcgen05 pipe of one thread executes in order).
//
// Softmax per block: one thread per row reads its 128 scores from TMEM,
// masks the diagonal block (warp-uniform branch), takes the row max, and
// keeps a lazily rescaled running max (O and the row sum are rescaled only
// when a row grows by more than 2^lazy_thresh).  The exp2 of the four 32-key
// chunks runs interleaved: MUFU for most, the FMA-pipe polynomial for the
// POLY chunks of unmasked blocks, so one warp keeps both pipes busy.
// ---------------------------------------------------------------------------
struct SmemPP {
  static constexpr int SLOTS = KV_SLOTS;
  static constexpr int Q = 0;                        // two Q tiles
  static constexpr int KV = Q + 2 * TILE_BYTES;
  static constexpr int BAR = KV + SLOTS * TILE_BYTES;
  // q full, q empty, full[SLOTS], empty[SLOTS], per tile: sfull, pfull (two
  // key halves), pvdone
  static constexpr int NBAR = 2 + 2 * SLOTS + 8;
  static constexpr int TMEM_PTR = BAR + NBAR * 8;
  static constexpr int TOTAL = TMEM_PTR + 16;
};

// Work unit `u` of the longest-first order: query-block pair and kv head.
struct Unit {
  int qb0, g, nb, maxpos;
};
__device__ __forceinline__ Unit unit_of(const Params& p, int u) {
  const int n_pairs = (p.n_qblocks + 1) / 2;
  Unit w;
  w.qb0 = (n_pairs - 1 - u / p.Hkv) * 2;
  w.g = u % p.Hkv;
  int maxpos = 0;
  for (int i = 0; i < 2 * p.QB; ++i) {
    const int a = w.qb0 * p.QB + i;
    if (a < p.A) maxpos = max(maxpos, __ldg(p.qpos + a));
  }
  w.maxpos = min(maxpos, p.n_ctx - 1);
  w.nb = w.maxpos / BLK_N + 1;
  return w;
}
// i-th unit of CTA c: rounds of gridDim.x units, alternate rounds reversed
__device__ __forceinline__ int unit_index(int i, int c, int grid) {
  return i * grid + ((i & 1) ? grid - 1 - c : c);
}

// P of 64 keys of a row (two 32-key chunks): element pair t of chunk c ->
// 2^(s*scale - m) via MUFU, or via the FMA-pipe polynomial when bit c of POLY
// is set; bf16x2 into pk[16c + t]; row sums per chunk (two FADD2 lanes
// each), added in chunk order.
template <uint32_t POLY>
__device__ __forceinline__ float p_half(const uint32_t* r, uint64_t sc2, uint64_t nm2,
                                        uint32_t* pk) {
  uint64_t acc[2][2];
#pragma unroll
  for (int c = 0; c < 2; ++c) acc[c][0] = acc[c][1] = pk2(0.f, 0.f);
#pragma unroll
  for (int t = 0; t < 16; ++t) {
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int i = 32 * c + 2 * t;
      const uint64_t a2 = ffma2(pk2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])), sc2, nm2);
      uint32_t e0, e1;
      if ((POLY >> c) & 1) {
        exp2_poly2(a2, e0, e1);
      } else {
        float a, b;
        upk2(a2, a, b);
        e0 = __float_as_uint(ex2(a));
        e1 = __float_as_uint(ex2(b));
      }
      acc[c][t & 1] = fadd2(acc[c][t & 1], (uint64_t)e0 | ((uint64_t)e1 << 32));
      pk[16 * c + t] = pack_bf16(__uint_as_float(e0), __uint_as_float(e1));
    }
  }
  float sum = 0.f;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    float s0, s1, s2, s3;
    upk2(acc[c][0], s0, s1);
    upk2(acc[c][1], s2, s3);
    sum += (s0 + s1) + (s2 + s3);
  }
  return sum;
}

template <uint32_t POLY_MASK>
__global__ void __launch_bounds__(32 * 10, 1)
attention_pp_kernel(const __grid_constant__ CUtensorMap map_q,
                    const __grid_constant__ CUtensorMap map_k,
                    const __grid_constant__ CUtensorMap map_v, const Params p) {
  using SM = SmemPP;
  constexpr int TMA_WARP = 8, MMA_WARP = 9;
  constexpr int NSLOT = SM::SLOTS;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sQ = base + SM::Q, sKV = base + SM::KV;
  const uint32_t bar0 = base + SM::BAR;
  const uint32_t bar_q = bar0, bar_qempty = bar0 + 8;
  auto bar_full = [&](int s) { return bar0 + (2 + s) * 8; };
  auto bar_empty = [&](int s) { return bar0 + (2 + NSLOT + s) * 8; };
  constexpr int B2 = 2 + 2 * NSLOT;
  auto bar_sfull = [&](int x) { return bar0 + (B2 + x) * 8; };
  // P of keys [64h, 64h+64) of tile x stored (h = 0, 1)
  auto bar_pfull = [&](int x, int h) { return bar0 + (B2 + 2 + 2 * x + h) * 8; };
  auto bar_pvdone = [&](int x) { return bar0 + (B2 + 6 + x) * 8; };
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(gbase + SM::TMEM_PTR);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n_units = ((p.n_qblocks + 1) / 2) * p.Hkv;
  const int grid = (int)gridDim.x, cta = (int)blockIdx.x;

  if (threadIdx.x == 0) {
    mbar_init(bar_q, 1);
    mbar_init(bar_qempty, 1);
    for (int s = 0; s < NSLOT; ++s) {
      mbar_init(bar_full(s), 1);
      mbar_init(bar_empty(s), 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(bar_sfull(x), 1);
      mbar_init(bar_pfull(x, 0), 4);  // one elected arrive per softmax warp of the tile
      mbar_init(bar_pfull(x, 1), 4);
      mbar_init(bar_pvdone(x), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_ptr)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_ptr;
  auto tS = [&](int x) { return tbase + (uint32_t)(x * 128); };
  auto tO = [&](int x) { return tbase + 256u + (uint32_t)(x * 128); };

  if (warp == TMA_WARP) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int slot = 0, i_unit = 0;
      uint32_t phase = 0;
      (void)i_unit;
      auto load = [&](const CUtensorMap* m, int g, int j, int tr) {
        mbar_wait(bar_empty(slot), phase ^ 1);
        CT_TRACE(6, tr, j, i_unit == 0);
        const uint32_t dst = sKV + slot * TILE_BYTES;
        mbar_expect_tx(bar_full(slot), TILE_BYTES);
        tma_load_3d(dst, m, bar_full(slot), 0, g, j * BLK_N);
        tma_load_3d(dst + ATOM_BYTES, m, bar_full(slot), 64, g, j * BLK_N);
        if (++slot == NSLOT) { slot = 0; phase ^= 1; }
      };
      for (int i = 0;; ++i) {
        const int u = unit_index(i, cta, grid);
        if (u >= n_units) break;
        const Unit w = unit_of(p, u);
        i_unit = i;
        // Q of this unit once the previous unit's last S MMA has read Q
        mbar_wait(bar_qempty, (uint32_t)((i & 1) ^ 1));
        mbar_expect_tx(bar_q, 2 * TILE_BYTES);
        for (int x = 0; x < 2; ++x) {
          const int a0 = (w.qb0 + x) * p.QB;
          tma_load_3d(sQ + x * TILE_BYTES, &map_q, bar_q, 0, w.g * p.G, a0);
          tma_load_3d(sQ + x * TILE_BYTES + ATOM_BYTES, &map_q, bar_q, 64, w.g * p.G, a0);
        }
        for (int j = 0; j < w.nb; ++j) {  // consumption order: K0 V0 K1 V1 ...
          load(&map_k, w.g, j, 0);
          load(&map_v, w.g, j, 1);
        }
      }
    }
  } else if (warp == MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t IDESC_S = idesc_bf16(false);
      constexpr uint32_t IDESC_O = idesc_bf16(true);
      int ring = 0;   // K/V ring position (2 per block)
      int gb = 0;     // blocks issued so far (both tiles), for barrier parities
      for (int i = 0;; ++i) {
        const int u = unit_index(i, cta, grid);
        if (u >= n_units) break;
        const int nb = unit_of(p, u).nb;
        mbar_wait(bar_q, (uint32_t)(i & 1));
        tc_fence_after();
        auto issue_s = [&](int x, int j) {
          const int ri = ring + 2 * j, s = ri % NSLOT;
          if (x == 0) {
            mbar_wait(bar_full(s), (uint32_t)((ri / NSLOT) & 1));
            tc_fence_after();
          }
          const uint64_t qd = sdesc(sQ + x * TILE_BYTES, 16, 1024);
          const uint64_t kd = sdesc(sKV + s * TILE_BYTES, 16, 1024);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t off16 = ((kk >> 2) * ATOM_BYTES + (kk & 3) * 32) >> 4;
            tc_mma(tS(x), qd + off16, kd + off16, IDESC_S, kk > 0);
          }
          if (x == 1) {
            tc_commit(bar_empty(s));
            if (j == nb - 1) tc_commit(bar_qempty);  // Q fully read: next unit's Q may land
          }
          tc_commit(bar_sfull(x));
          CT_TRACE(3, x, j, i == 0);
        };
        auto issue_pv = [&](int x, int j) {
          const int ri = ring + 2 * j + 1, s = ri % NSLOT;
          const uint32_t par = (uint32_t)((gb + j) & 1);
          CT_TRACE(5, x, j, i == 0);
          if (x == 0) mbar_wait(bar_full(s), (uint32_t)((ri / NSLOT) & 1));
          CT_TRACE(12, x, j, i == 0);
          const uint64_t vd = sdesc(sKV + s * TILE_BYTES, ATOM_BYTES, 1024);
          // the first key half's PV runs while the softmax finishes the second
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            mbar_wait(bar_pfull(x, h), par);
            tc_fence_after();
            if (h == 0) CT_TRACE(2, x, j, i == 0);
#pragma unroll
            for (int kk = 4 * h; kk < 4 * h + 4; ++kk)
              // A = P_x: keys [16kk, 16kk+16) = bf16x2 TMEM columns [8kk, 8kk+8)
              tc_mma_ts(tO(x), tS(x) + kk * 8, vd + (uint64_t)(kk * 2048 / 16), IDESC_O,
                        (j > 0 || kk > 0) ? 1u : 0u);
          }
          if (x == 1) tc_commit(bar_empty(s));
          tc_commit(bar_pvdone(x));
        };
        issue_s(0, 0);
        issue_s(1, 0);
        for (int j = 0; j < nb; ++j) {
          issue_pv(0, j);
          if (j + 1 < nb) issue_s(0, j + 1);
          issue_pv(1, j);
          if (j + 1 < nb) issue_s(1, j + 1);
        }
        ring += 2 * nb;
        gb += nb;
      }
    }
  } else {
    // ------------------------------------------------------------ softmax
    const int x = warp / 4;                   // tile
    const int m = (warp & 3) * 32 + lane;     // TMEM lane / tile row
    const int qi = m / p.G, hj = m % p.G;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint64_t sc2 = pk2(p.scale_log2, p.scale_log2);
    int gb = 0;
    for (int i = 0;; ++i) {
      const int u = unit_index(i, cta, grid);
      if (u >= n_units) break;
      const Unit w = unit_of(p, u);
      const int a = (w.qb0 + x) * p.QB + qi;
      const bool valid = a < p.A;
      const int pos = valid ? min(__ldg(p.qpos + a), p.n_ctx - 1) : w.maxpos;
      float m_used = -INFINITY, l = 0.f;
      uint32_t r[BLK_N];
      for (int j = 0; j < w.nb; ++j) {
        const uint32_t par = (uint32_t)((gb + j) & 1);
        mbar_wait(bar_sfull(x), par);
        __syncwarp();
        tc_fence_after();
        CT_TRACE(0, x, j, i == 0 && (warp & 3) == 0 && lane == 0);
        const int kbase = j * BLK_N;
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_ld32(tS(x) + lane_off + 32 * c, r + 32 * c);
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_wait_ld32(r + 32 * c);
        // the diagonal block(s) of a row: keys past its position -> -inf.
        // Warp-uniform branch (no divergence); such blocks stay all-MUFU so
        // masked keys give exactly 0.
        const bool masked = __any_sync(0xffffffffu, kbase + BLK_N - 1 > pos);
        if (masked) {
#pragma unroll
          for (int c = 0; c < BLK_N; ++c)
            if (kbase + c > pos) r[c] = __float_as_uint(-INFINITY);
        }
        float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < BLK_N; c += 8) {
#pragma unroll
          for (int t = 0; t < 4; ++t)
            mq[t] = max3f(mq[t], __uint_as_float(r[c + 2 * t]), __uint_as_float(r[c + 2 * t + 1]));
        }
        const float mx = max3f(mq[0], mq[1], fmaxf(mq[2], mq[3])) * p.scale_log2;
        const float m_new = fmaxf(m_used, mx);
        const bool grow = m_new > m_used + p.lazy_thresh;
        const bool any_grow = __any_sync(0xffffffffu, grow);
        const float corr = grow ? ex2(m_used - m_new) : 1.f;  // 0 when m_used = -inf
        if (grow) m_used = m_new;
        const uint64_t nm2 = pk2(-m_used, -m_used);
        // P = 2^(s*scale - m): the four 32-key chunks advance in lockstep so
        // the MUFU exp2 of three chunks and the FMA-pipe polynomial exp2 of
        // the POLY chunk (unmasked blocks) issue interleaved from one warp,
        // with the argument FFMA2s, bf16 packing and FADD2 row sums in the
        // gaps of the 8-cycle MUFU issue.
        if (any_grow && j > 0) {
          // O_x *= corr once PV_x(j-1) has landed (warp-uniform branch)
          mbar_wait(bar_pvdone(x), (uint32_t)((gb + j - 1) & 1));
          __syncwarp();
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < HD / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(tO(x) + lane_off + c * 32, o);
            tmem_wait_ld32(o);
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
            tmem_st32(tO(x) + lane_off + c * 32, o);
          }
          tmem_wait_st();
        }
        // P in two key halves: the MMA warp starts PV on keys [0, 64) while
        // this warp exponentiates keys [64, 128)
        float bsum = 0.f;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t pk[32];
          if (masked || POLY_MASK == 0)
            bsum += p_half<0u>(r + 64 * h, sc2, nm2, pk);
          else if (h == 0)
            bsum += p_half<POLY_MASK & 3u>(r, sc2, nm2, pk);
          else
            bsum += p_half<(POLY_MASK >> 2) & 3u>(r + 64, sc2, nm2, pk);
          tmem_st16(tS(x) + lane_off + 32 * h, pk);
          tmem_st16(tS(x) + lane_off + 32 * h + 16, pk + 16);
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          CT_TRACE(h == 1 ? 1 : 4, x, j, i == 0 && (warp & 3) == 0 && lane == 0);
          CT_TRACE(8 + (warp & 3), x, j, h == 0 && i == 0 && lane == 0);
          if (lane == 0) mbar_arrive(bar_pfull(x, h));
          if (h == 0) {
            // Re-read keys [64, 128) (their S columns are never overwritten by
            // P): the true dependency keeps the second half's exp2 behind the
            // first half's hand-off, which the scheduler would otherwise sink
            // below all the MUFU work.
            tmem_ld32(tS(x) + lane_off + 64, r + 64);
            tmem_ld32(tS(x) + lane_off + 96, r + 96);
            tmem_wait_ld32(r + 64);
            tmem_wait_ld32(r + 96);
            if (masked) {
#pragma unroll
              for (int c = 64; c < BLK_N; ++c)
                if (kbase + c > pos) r[c] = __float_as_uint(-INFINITY);
            }
          }
        }
        l = l * corr + bsum;
      }
      // epilogue: O_x / l -> global once PV_x(nb-1) has landed
      mbar_wait(bar_pvdone(x), (uint32_t)((gb + w.nb - 1) & 1));
      __syncwarp();
      tc_fence_after();
      const float inv = valid ? 1.f / l : 0.f;
      const int64_t orow = ((int64_t)a * p.Hq + (int64_t)w.g * p.G + hj) * HD;
#pragma unroll 1
      for (int c = 0; c < HD / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tO(x) + lane_off + c * 32, o);
        tmem_wait_ld32(o);
        if (valid) {
          if (p.out_f32) {
            float4* dst = reinterpret_cast<float4*>(p.out_f32 + orow + c * 32);
#pragma unroll
            for (int e = 0; e < 8; ++e)
              dst[e] = make_float4(__uint_as_float(o[4 * e]) * inv, __uint_as_float(o[4 * e + 1]) * inv,
                                   __uint_as_float(o[4 * e + 2]) * inv, __uint_as_float(o[4 * e + 3]) * inv);
          } else {
            uint4* dst = reinterpret_cast<uint4*>(p.out + orow + c * 32);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              uint4 v;
              v.x = pack_bf16(__uint_as_float(o[8 * e + 0]) * inv, __uint_as_float(o[8 * e + 1]) * inv);
              v.y = pack_bf16(__uint_as_float(o[8 * e + 2]) * inv, __uint_as_float(o[8 * e + 3]) * inv);
              v.z = pack_bf16(__uint_as_float(o[8 * e + 4]) * inv, __uint_as_float(o[8 * e + 5]) * inv);
              v.w = pack_bf16(__uint_as_float(o[8 * e + 6]) * inv, __uint_as_float(o[8 * e + 7]) * inv);
              dst[e] = v;
            }
          }
        }
      }
      // the O reads above precede this warp's first pfull arrive of the next
      // unit, which the PV that overwrites O_x (accumulate = 0) waits for
      gb += w.nb;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512)
                 : "memory");
  }
}

using EncodeFn = PFN_cuTensorMapEncodeTiled_v12000;

static EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeFn)p;
  }
  return fn;
}

static int make_map(CUtensorMap* map, const void* ptr, uint64_t d1, uint64_t d2,
                    uint64_t stride1_bytes, uint64_t stride2_bytes, uint32_t box1, uint32_t box2) {
  EncodeFn enc = encode_fn();
  if (!enc) return fail(CT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {HD, d1, d2};
  cuuint64_t strides[2] = {stride1_bytes, stride2_bytes};
  cuuint32_t box[3] = {64, box1, box2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CT_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return CT_OK;
}

// Process-wide knobs, read once.  CT_TC_LAZY: rescale threshold (log2 units,
// default 8); CT_TC_POLY=<0,1,2,4,5,8>: which of
// the four 32-key chunks of a block take the FMA-pipe exp2 (all values are
// correct; 0 = all MUFU).
struct TcKnobs {
  float lazy = LAZY_THRESH;
  int poly = 0;
  TcKnobs() {
    if (const char* e = getenv("CT_TC_LAZY")) lazy = (float)atof(e);
    if (const char* e = getenv("CT_TC_POLY")) poly = (int)strtol(e, nullptr, 0) & 15;
  }
};
static const TcKnobs& knobs() {
  static const TcKnobs k;
  return k;
}

static int sm_count() {
  static int n = [] {
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

}  // namespace tc

// tcgen05 preconditions: D = 128, GQA group divides the 128-row tile, 16-byte
// aligned operands and rows (TMA).  Otherwise the SIMT kernel runs.
bool tc_supported(const void* q, const void* k_cache, const void* v_cache, int64_t Hq,
                  int64_t Hkv, int64_t D, int64_t cache_row_stride) {
  if (D != tc::HD || Hkv < 1 || Hq % Hkv) return false;
  const int64_t G = Hq / Hkv;
  if (G < 1 || tc::TILE_M % G) return false;
  if (((uintptr_t)q | (uintptr_t)k_cache | (uintptr_t)v_cache) & 15) return false;
  return (cache_row_stride * 2) % 16 == 0;
}

size_t attention_tc_workspace(int64_t, int64_t, int64_t, int64_t, int64_t) { return 0; }

int attention_tc(const void* q, const int32_t* q_pos, int64_t A, int64_t Hq, const void* k_cache,
                 const void* v_cache, int64_t n_ctx, int64_t Hkv, int64_t D,
                 int64_t cache_row_stride, double scale, void* out, int out_dtype,
                 void* workspace, size_t workspace_bytes, cudaStream_t st) {
  using namespace tc;
  (void)workspace;
  (void)workspace_bytes;
  if (!tc_supported(q, k_cache, v_cache, Hq, Hkv, D, cache_row_stride))
    return fail(CT_ERR_UNSUPPORTED, "tcgen05 attention preconditions not met");
  const int64_t G = Hq / Hkv;
  CUtensorMap mq, mk, mv;
  int rc;
  if ((rc = make_map(&mq, q, (uint64_t)Hq, (uint64_t)A, HD * 2, (uint64_t)Hq * HD * 2,
                     (uint32_t)G, (uint32_t)(TILE_M / G))))
    return rc;
  if ((rc = make_map(&mk, k_cache, (uint64_t)Hkv, (uint64_t)n_ctx, HD * 2,
                     (uint64_t)cache_row_stride * 2, 1, BLK_N)))
    return rc;
  if ((rc = make_map(&mv, v_cache, (uint64_t)Hkv, (uint64_t)n_ctx, HD * 2,
                     (uint64_t)cache_row_stride * 2, 1, BLK_N)))
    return rc;
  const TcKnobs& kn = knobs();
  Params prm;
  prm.qpos = q_pos;
  prm.out = out_dtype == CT_BF16 ? (__nv_bfloat16*)out : nullptr;
  prm.out_f32 = out_dtype == CT_F32 ? (float*)out : nullptr;
  prm.A = (int)A;
  prm.Hq = (int)Hq;
  prm.Hkv = (int)Hkv;
  prm.G = (int)G;
  prm.QB = (int)(TILE_M / G);
  prm.n_ctx = (int)n_ctx;
  prm.n_qblocks = (int)((A + prm.QB - 1) / prm.QB);
  prm.scale_log2 = (float)(scale * 1.4426950408889634);
  prm.lazy_thresh = kn.lazy;
  using KernFn = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, Params);
  KernFn kp;
  switch (kn.poly) {
    case 0: kp = attention_pp_kernel<0u>; break;
    case 1: kp = attention_pp_kernel<1u>; break;
    case 2: kp = attention_pp_kernel<2u>; break;
    case 4: kp = attention_pp_kernel<4u>; break;
    case 8: kp = attention_pp_kernel<8u>; break;
    case 5: kp = attention_pp_kernel<5u>; break;
    default: return fail(CT_ERR_PARAM, "CT_TC_POLY=%d is not built (0, 1, 2, 4, 5, 8)", kn.poly);
  }
  const size_t smem = SmemPP::TOTAL + 1024;
  CT_CUDA(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int n_units = ((prm.n_qblocks + 1) / 2) * prm.Hkv;
  const unsigned grid = (unsigned)std::min(n_units, sm_count());
  kp<<<grid, 32 * 10, smem, st>>>(mq, mk, mv, prm);
#ifdef CT_ATT_TRACE
  if (const char* path = getenv("CT_TC_TRACE_OUT")) {
    static unsigned long long h[14][2][512];
    cudaStreamSynchronize(st);
    cudaMemcpyFromSymbol(h, g_trace, sizeof(h));
    if (FILE* f = fopen(path, "w")) {
      for (int j = 0; j < 512; ++j)
        for (int x = 0; x < 2; ++x) {
          fprintf(f, "%d %d ", j, x);
          for (int e = 0; e < 14; ++e) fprintf(f, "%s%llu", e ? " " : "", h[e][x][j]);
          fprintf(f, "\n");
        }
      fclose(f);
    }
  }
#endif
  return check_launch("attention_pp_kernel");
}

}  // namespace ct
