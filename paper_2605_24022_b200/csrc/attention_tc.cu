// (4) Selective-recompute attention on the 5th-gen tensor cores (sm_100a):
// tcgen05.mma with fp32 accumulators in TMEM, bf16 operands staged by TMA.
// Replaces the attention of ct/toymodel.py:176-183 (q = selected rows + suffix
// at global positions, keys/values = the full blended cache, key j visible to
// a query iff j <= its position).
//
// Tile = 128 TMEM lanes = (128/G queries) x (G q-heads of one kv-head), so a
// K/V tile staged once serves the whole GQA group.  Per 128-key block:
//   S = Q K^T      tcgen05.mma  M128 N128 K16 x8, A=Q smem, B=K smem -> TMEM
//   softmax        one thread per row: tcgen05.ld S row, mask by position,
//                  exp2, lazy max (rescale O only when the max grows > 2^8),
//                  P (bf16) written swizzled to smem
//   O += P V       tcgen05.mma  M128 N128 K16 x8, A=P smem, B=V smem (MN-major)
// Warp roles: warps 0-7 softmax/epilogue (two warps per TMEM lane quarter,
// each owning half of the key columns), warp 8 TMA producer, warp 9 MMA
// issuer (+TMEM alloc).  S is double buffered in TMEM,
// P double buffered in smem, K/V flow through a 3-slot TMA ring.
#include "common.cuh"

#include <cuda.h>
#include <type_traits>
#include <cudaTypedefs.h>

// The timing-probe schedules (SCHED 3/4) end the softmax loop body with
// `continue`, which makes the rest of the body unreachable in those
// instantiations only.
#pragma nv_diag_suppress 128

namespace ct {

namespace tc {

constexpr int TILE_M = 128;   // TMEM lanes / MMA M
constexpr int BLK_N = 128;    // keys per block
constexpr int HD = 128;       // head dim
constexpr int KV_SLOTS = 5;
constexpr int MAX_SPLIT = 4;         // softmax threads per tile row (key-column split)
constexpr int NSB = 3;               // S/P TMEM buffers
constexpr int ATOM_BYTES = 128 * 64 * 2;      // [128 rows][64 bf16] swizzle-128B half tile
constexpr int TILE_BYTES = 2 * ATOM_BYTES;    // 32 KiB: 128 rows x 128 bf16
constexpr float LAZY_THRESH = 8.0f;           // log2 units

// CTAS = 1: one CTA owns a 128-row tile and stages whole K/V tiles (32 KiB).
// CTAS = 2: a CTA pair (cluster of 2, tcgen05 cta_group::2, MMA M = 256)
// owns two 128-row tiles; each CTA stages HALF of every K tile (64 keys) and
// half of every V tile (64 head-dim columns), 16 KiB per slot, so per SM the
// K/V bytes from L2 and the MMA operand reads from shared memory halve.
template <int CTAS>
struct Smem {
  static constexpr int SLOT_BYTES = TILE_BYTES / CTAS;
  static constexpr int SLOTS = CTAS == 1 ? KV_SLOTS : 2 * KV_SLOTS;
  // offsets from the 1024-aligned base
  static constexpr int Q = 0;
  static constexpr int KV = Q + TILE_BYTES;
  static constexpr int BAR = KV + SLOTS * SLOT_BYTES;
  // q + KV full/empty + per S/P buffer (S full, P full, PV done); the
  // exchange area must not overlap the last barrier
  static constexpr int NBAR = 1 + 2 * SLOTS + 3 * 3;
  static constexpr int XCH = BAR + NBAR * 8;  // [3][MAX_SPLIT][128] f32 max/sum exchange
  static constexpr int TMEM_PTR = XCH + 3 * MAX_SPLIT * 128 * 4;
  static constexpr int TOTAL = TMEM_PTR + 16;
};

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
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
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
// 2-SM TMA: bytes land in this CTA's smem, completion counts on the LEADER's
// mbarrier (same offset, peer bit cleared).
__device__ __forceinline__ void tma_load_3d_2sm(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                                int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(map), "r"(bar & 0xFEFFFFFFu), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same smem offset in CTA `rank`
__device__ __forceinline__ uint32_t mapa_rank(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "LAB_WAITC:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONEC;\n\t"
      "bra LAB_WAITC;\n\t"
      "DONEC:\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
template <int CTAS>
__device__ __forceinline__ void tc_commit_t(uint32_t bar) {
  if constexpr (CTAS == 1) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], m;\n\t}" ::"r"(bar)
        : "memory");
  }
}
template <int CTAS>
__device__ __forceinline__ void tc_mma_t(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accum) {
  if constexpr (CTAS == 1) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
  }
}
template <int CTAS>
__device__ __forceinline__ void tc_mma_ts_t(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                            uint32_t idesc, uint32_t accum) {
  if constexpr (CTAS == 1) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accum)
        : "memory");
  }
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
// Which of a thread's 8 chunks of 8 scores take the FMA-pipe polynomial
// instead of MUFU.ex2 (template parameter; 0 = all MUFU).

// p = 2^(s*scale - m) for the thread's HALF scores: packed FFMA2 for the
// argument, MUFU.ex2 or the polynomial per chunk (compile-time POLY), FADD2
// row-sum accumulators, bf16x2 packing for the TMEM P store.
__device__ __forceinline__ uint32_t pack_bf16(float a, float b);

template <int HALF, uint32_t POLY>
__device__ __forceinline__ void softmax_chunks(const uint32_t* r, uint64_t sc2, uint64_t nm2,
                                               uint64_t* acc2, uint32_t* pk) {
#pragma unroll
  for (int ch = 0; ch < HALF / 8; ++ch) {
    uint64_t x2[4];
#pragma unroll
    for (int t = 0; t < 4; ++t)
      x2[t] = ffma2(pk2(__uint_as_float(r[ch * 8 + 2 * t]), __uint_as_float(r[ch * 8 + 2 * t + 1])),
                    sc2, nm2);
    uint32_t e[8];
    if (((POLY >> (ch & 31)) & 1) != 0) {  // folds per unrolled chunk
#pragma unroll
      for (int t = 0; t < 4; ++t) exp2_poly2(x2[t], e[2 * t], e[2 * t + 1]);
    } else {
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        float x0, x1;
        upk2(x2[t], x0, x1);
        e[2 * t] = __float_as_uint(ex2(x0));
        e[2 * t + 1] = __float_as_uint(ex2(x1));
      }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
      acc2[t & 1] = fadd2(acc2[t & 1], (uint64_t)e[2 * t] | ((uint64_t)e[2 * t + 1] << 32));
#pragma unroll
    for (int t = 0; t < 4; ++t)
      pk[ch * 4 + t] = pack_bf16(__uint_as_float(e[2 * t]), __uint_as_float(e[2 * t + 1]));
  }
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

template <int NSPLIT, uint32_t POLY_MASK, int EXPT = 0, int CTAS = 1>
__global__ void __launch_bounds__(32 * (4 * NSPLIT + 2), 1)
attention_tc_kernel(const __grid_constant__ CUtensorMap map_q,
                    const __grid_constant__ CUtensorMap map_k,
                    const __grid_constant__ CUtensorMap map_v, const Params p) {
  constexpr int SOFTMAX_WARPS = 4 * NSPLIT;
  constexpr int TMA_WARP = SOFTMAX_WARPS, MMA_WARP = SOFTMAX_WARPS + 1;
  constexpr int HALF = BLK_N / NSPLIT;  // key columns per softmax thread
  constexpr int NSM = 32 * SOFTMAX_WARPS;
  using SM = Smem<CTAS>;
  constexpr int NSLOT = SM::SLOTS;
  constexpr int SLOT = SM::SLOT_BYTES;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sQ = base + SM::Q, sKV = base + SM::KV;
  const uint32_t bar0 = base + SM::BAR;
  const uint32_t crank = CTAS == 2 ? cluster_rank() : 0u;
  const bool leader = crank == 0;
  // barriers
  const uint32_t bar_q = bar0 + 0 * 8;
  auto bar_full = [&](int s) { return bar0 + (1 + s) * 8; };
  auto bar_empty = [&](int s) { return bar0 + (1 + NSLOT + s) * 8; };
  constexpr int B2 = 1 + 2 * NSLOT;
  // per S/P TMEM buffer (3): S landed, P written, PV (the reader of P) done
  auto bar_sfull = [&](int b) { return bar0 + (B2 + b) * 8; };
  auto bar_pfull = [&](int b) { return bar0 + (B2 + 3 + b) * 8; };
  auto bar_pvdone = [&](int b) { return bar0 + (B2 + 6 + b) * 8; };
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(gbase + SM::TMEM_PTR);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // longest tiles first: high query blocks (largest positions) get low block
  // ids.  A CTA pair takes two adjacent query blocks of one kv head.
  const int tile = blockIdx.x / CTAS;
  const int n_units = (p.n_qblocks + CTAS - 1) / CTAS;
  const int qb0 = (n_units - 1 - (tile / p.Hkv)) * CTAS;
  const int qb = qb0 + (int)crank;
  const int g = tile % p.Hkv;
  const int a0 = qb * p.QB;

  // key range: the pair shares every K/V block, so both use the pair's max
  int maxpos = 0;
  for (int i = 0; i < CTAS * p.QB; ++i) {
    const int a = qb0 * p.QB + i;
    if (a < p.A) maxpos = max(maxpos, __ldg(p.qpos + a));
  }
  maxpos = min(maxpos, p.n_ctx - 1);
  const int nb = maxpos / BLK_N + 1;

  if (threadIdx.x == 0) {
    // full / q: the leader's copies count one arrive per CTA of the pair (the
    // leader's carries expect_tx for both CTAs' bytes); pfull: one elected
    // arrive per softmax warp of every CTA of the pair
    mbar_init(bar_q, CTAS);
    for (int s = 0; s < NSLOT; ++s) {
      mbar_init(bar_full(s), CTAS);
      mbar_init(bar_empty(s), 1);
    }
    for (int b = 0; b < NSB; ++b) {
      mbar_init(bar_sfull(b), 1);
      mbar_init(bar_pfull(b), (EXPT == 3 ? 1 : CTAS) * SOFTMAX_WARPS);
      mbar_init(bar_pvdone(b), 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == MMA_WARP) {
    if constexpr (CTAS == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       su32(tmem_ptr)),
                   "r"(512)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       su32(tmem_ptr)),
                   "r"(512)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if constexpr (CTAS == 2) cluster_sync_all();  // peer barriers initialised before any signal
  else __syncthreads();
  tc_fence_after();
  // leader-side copy of a barrier (remote for the peer CTA)
  auto to_leader = [&](uint32_t bar) { return CTAS == 2 ? mapa_rank(bar, 0) : bar; };
  auto arrive_tx = [&](uint32_t bar, uint32_t bytes) {
    if (leader) mbar_expect_tx(bar, bytes * CTAS);
    else mbar_arrive_cluster(to_leader(bar));
  };
  const uint32_t tbase = *tmem_ptr;
  // TMEM: three S buffers (128 fp32 columns each) + O (128).  P_j (bf16x2,
  // 64 columns) overwrites the first half of S_j's buffer once the softmax
  // has read S_j; the PV MMA reads it as its TMEM A operand, so P never
  // touches shared memory.  Three buffers let S run two blocks ahead.
  auto tS = [&](int b) { return tbase + (uint32_t)(b * 128); };
  const uint32_t tO = tbase + 384;

  if (warp == TMA_WARP) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      auto tma = [&](uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1, int c2) {
        if constexpr (CTAS == 1) tma_load_3d(dst, m, bar, c0, c1, c2);
        else tma_load_3d_2sm(dst, m, bar, c0, c1, c2);
      };
      arrive_tx(bar_q, TILE_BYTES);
      tma(sQ, &map_q, bar_q, 0, g * p.G, a0);
      tma(sQ + ATOM_BYTES, &map_q, bar_q, 64, g * p.G, a0);
      int slot = 0;
      uint32_t phase = 0;
      // K_j: CTAS=1 the whole [128 keys][128 d] tile (two 64-d swizzle atoms);
      // CTAS=2 keys [64r, 64r+64) of the block (MMA N half r), both d atoms.
      int nloads = 0;
      auto load_k = [&](int j) {
        mbar_wait(bar_empty(slot), phase ^ 1);
        const uint32_t dst = sKV + slot * SLOT;
        if (EXPT == 4 && ++nloads > NSLOT) {  // probe: slots keep stale data
          if (leader) mbar_arrive(bar_full(slot));
          else mbar_arrive_cluster(to_leader(bar_full(slot)));
          if (++slot == NSLOT) { slot = 0; phase ^= 1; }
          return;
        }
        arrive_tx(bar_full(slot), SLOT);
        const int key0 = j * BLK_N + (int)crank * (BLK_N / CTAS);
        tma(dst, &map_k, bar_full(slot), 0, g, key0);
        tma(dst + SLOT / 2, &map_k, bar_full(slot), 64, g, key0);
        if (++slot == NSLOT) { slot = 0; phase ^= 1; }
      };
      // V_j: CTAS=1 both 64-d atoms; CTAS=2 the d atom r (MMA N half r).
      auto load_v = [&](int j) {
        mbar_wait(bar_empty(slot), phase ^ 1);
        const uint32_t dst = sKV + slot * SLOT;
        if (EXPT == 4 && ++nloads > NSLOT) {
          if (leader) mbar_arrive(bar_full(slot));
          else mbar_arrive_cluster(to_leader(bar_full(slot)));
          if (++slot == NSLOT) { slot = 0; phase ^= 1; }
          return;
        }
        arrive_tx(bar_full(slot), SLOT);
        if constexpr (CTAS == 1) {
          tma(dst, &map_v, bar_full(slot), 0, g, j * BLK_N);
          tma(dst + ATOM_BYTES, &map_v, bar_full(slot), 64, g, j * BLK_N);
        } else {
          tma(dst, &map_v, bar_full(slot), 64 * (int)crank, g, j * BLK_N);
        }
        if (++slot == NSLOT) { slot = 0; phase ^= 1; }
      };
      // same order the MMA warp consumes: K0, K1, K2, V0, K3, V1, K4, ...
      for (int j = 0; j < NSB && j < nb; ++j) load_k(j);
      for (int j = 0; j < nb; ++j) {
        load_v(j);
        if (j + NSB < nb) load_k(j + NSB);
      }
    }
  } else if (warp == MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0 && leader) {
      constexpr uint32_t IDESC_S = idesc_bf16(false, TILE_M * CTAS);
      constexpr uint32_t IDESC_O = idesc_bf16(true, TILE_M * CTAS);
      constexpr int KATOM = SLOT / 2;  // bytes of one 64-d K atom in a slot
      mbar_wait(bar_q, 0);
      tc_fence_after();
      int slot = 0;
      uint32_t phase = 0;
      // S_j goes into TMEM buffer j%3, which last held P_{j-3}.  S_j is issued
      // right after PV_{j-3} (its reader) by this thread, and tcgen05.mma ops
      // from one thread execute in issue order, so no wait is needed: two S
      // blocks stay queued ahead of every PV while the softmax works.
      auto issue_s = [&](int j) {
        const int b = j % NSB;
        mbar_wait(bar_full(slot), phase);
        tc_fence_after();
        const uint32_t k_tile = sKV + slot * SLOT;
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t koff = (kk & 3) * 32;
          tc_mma_t<CTAS>(tS(b), sdesc(sQ + (kk >> 2) * ATOM_BYTES + koff, 16, 1024),
                         sdesc(k_tile + (kk >> 2) * KATOM + koff, 16, 1024), IDESC_S, kk > 0);
        }
        tc_commit_t<CTAS>(bar_empty(slot));
        tc_commit_t<CTAS>(bar_sfull(b));
        if (++slot == NSLOT) { slot = 0; phase ^= 1; }
      };
      for (int j = 0; j < NSB && j < nb; ++j) issue_s(j);
      for (int j = 0; j < nb; ++j) {
        // O += P_j V_j
        const int b = j % NSB;
        if constexpr (CTAS == 2) mbar_wait_cluster(bar_pfull(b), (j / NSB) & 1);
        else mbar_wait(bar_pfull(b), (j / NSB) & 1);
        mbar_wait(bar_full(slot), phase);
        tc_fence_after();
        const uint32_t v_tile = sKV + slot * SLOT;
#pragma unroll
        for (int kk = 0; kk < BLK_N / 16; ++kk) {
          // A = P from TMEM (16 keys = 8 packed columns); B = V, MN-major,
          // K-step of 16 keys = 2 x 1024 B core-matrix groups
          tc_mma_ts_t<CTAS>(tO, tS(b) + kk * 8, sdesc(v_tile + kk * 2048, ATOM_BYTES, 1024),
                            IDESC_O, (j > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit_t<CTAS>(bar_empty(slot));
        tc_commit_t<CTAS>(bar_pvdone(b));
        if (++slot == NSLOT) { slot = 0; phase ^= 1; }
        if (j + NSB < nb) issue_s(j + NSB);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax
    // 8 warps: warp w owns TMEM lanes 32*(w%4).. (tile rows) and the column
    // half hf = w/4 (keys 64*hf .. +63 of each block, O columns likewise), so
    // every SMSP runs two softmax warps.  The two halves of a row agree on the
    // running max through a double-buffered smem exchange + named barrier.
    const int hf = warp >> 2;
    const int m = (warp & 3) * 32 + lane;  // TMEM lane / tile row
    const int qi = m / p.G, hj = m % p.G;
    const int a = a0 + qi;
    const bool valid = a < p.A;
    const int pos = valid ? min(__ldg(p.qpos + a), p.n_ctx - 1) : maxpos;
    const uint32_t lane_off = ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(hf * HALF);
    const uint32_t lane_off_p = ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(hf * HALF / 2);
    float* xch = reinterpret_cast<float*>(gbase + SM::XCH);  // [3][2][128]
    float m_used = -INFINITY, l = 0.f;
    uint32_t r[HALF];
    for (int j = 0; j < nb; ++j) {
      const int b = j % NSB;
      mbar_wait(bar_sfull(b), (j / NSB) & 1);
      // lanes leave the try_wait spin independently: reconverge before the
      // warp-collective (.sync.aligned) tcgen05.ld
      __syncwarp();
      tc_fence_after();
      if constexpr (EXPT == 2 || EXPT == 3 || EXPT == 4) {  // profiling aid: no softmax
        tc_fence_before();
        __syncwarp();
        if (EXPT == 3 && !leader) continue;  // EXPT 3: leader does not wait for the peer
        if (lane == 0) {
          if constexpr (CTAS == 2) mbar_arrive_cluster(to_leader(bar_pfull(b)));
          else mbar_arrive(bar_pfull(b));
        }
        continue;
      }
      if constexpr (EXPT == 1) {  // profiling aid: TMEM S load + P store only
#pragma unroll
        for (int c = 0; c < HALF / 32; ++c) tmem_ld32(tS(b) + lane_off + c * 32, r + c * 32);
#pragma unroll
        for (int c = 0; c < HALF / 32; ++c) tmem_wait_ld32(r + c * 32);
        uint32_t pk[HALF / 2];
#pragma unroll
        for (int c = 0; c < HALF / 2; ++c) pk[c] = r[2 * c] ^ r[2 * c + 1];
        asm volatile("bar.sync 1, %0;" ::"n"(NSM) : "memory");
        __syncwarp();
#pragma unroll
        for (int c = 0; c < HALF / 64; ++c) tmem_st32(tS(b) + lane_off_p + c * 32, pk + c * 32);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if constexpr (CTAS == 2) mbar_arrive_cluster(to_leader(bar_pfull(b)));
          else mbar_arrive(bar_pfull(b));
        }
        continue;
      }
#pragma unroll
      for (int c = 0; c < HALF / 32; ++c) tmem_ld32(tS(b) + lane_off + c * 32, r + c * 32);
#pragma unroll
      for (int c = 0; c < HALF / 32; ++c) tmem_wait_ld32(r + c * 32);
      const int kbase = j * BLK_N + hf * HALF;
      const bool need_mask = kbase + HALF - 1 > pos;
      if (need_mask) {
#pragma unroll
        for (int c = 0; c < HALF; ++c)
          if (kbase + c > pos) r[c] = __float_as_uint(-INFINITY);
      }
      // row max of the raw scores (scale > 0 commutes with max)
      float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < HALF; c += 8) {
#pragma unroll
        for (int t = 0; t < 4; ++t)
          mq[t] = max3f(mq[t], __uint_as_float(r[c + 2 * t]), __uint_as_float(r[c + 2 * t + 1]));
      }
      const float pm = max3f(mq[0], mq[1], fmaxf(mq[2], mq[3]));
      float* xb = xch + (j & 1) * (NSPLIT * 128);
      float mrow = pm;
      if constexpr (NSPLIT > 1) {
        xb[hf * 128 + m] = pm;
        // also orders every half's S_j reads before any half's P_j writes
        // (P_j aliases the first half of S_j's TMEM columns)
        tc_fence_before();
        asm volatile("bar.sync 1, %0;" ::"n"(NSM) : "memory");
        tc_fence_after();
#pragma unroll
        for (int o = 1; o < NSPLIT; ++o) mrow = fmaxf(mrow, xb[((hf + o) % NSPLIT) * 128 + m]);
      }
      const float mx = mrow * p.scale_log2;
      const float m_new = fmaxf(m_used, mx);
      const bool grow = m_new > m_used + p.lazy_thresh;
      // warp-uniform decision (tcgen05.ld/st are .sync.aligned).  P_j is built
      // with the new max first; the O rescale (which must wait for PV_{j-1})
      // runs after P_j is in smem so it overlaps PV_{j-1} instead of stalling.
      const bool any_grow = __any_sync(0xffffffffu, grow);
      const float corr = grow ? ex2(m_used - m_new) : 1.f;  // 0 when m_used = -inf
      if (grow) m_used = m_new;
      // P_j half-row into smem buffer b: atom hf (K-major SW128, chunk c^(m&7))
      uint32_t pk[HALF / 2];  // packed bf16x2 P for this thread's key columns
      const uint64_t sc2 = pk2(p.scale_log2, p.scale_log2);
      const uint64_t nm2 = pk2(-m_used, -m_used);
      uint64_t acc2[2] = {pk2(0.f, 0.f), pk2(0.f, 0.f)};
      // masked (diagonal) blocks take the all-MUFU path: -inf must give 0
      if (need_mask)
        softmax_chunks<HALF, 0u>(r, sc2, nm2, acc2, pk);
      else
        softmax_chunks<HALF, POLY_MASK>(r, sc2, nm2, acc2, pk);
      {
        float s0, s1, s2, s3;
        upk2(acc2[0], s0, s1);
        upk2(acc2[1], s2, s3);
        l = l * corr + ((s0 + s1) + (s2 + s3));  // partial row sum over this half
      }
      // P_j -> TMEM columns [hf*HALF/2, +HALF/2) of P buffer b (lane m)
      __syncwarp();
#pragma unroll
      for (int c = 0; c < HALF / 64; ++c) tmem_st32(tS(b) + lane_off_p + c * 32, pk + c * 32);
      if constexpr (HALF / 2 < 32) tmem_st16(tS(b) + lane_off_p, pk);
      tmem_wait_st();
      if (any_grow && j > 0) {
        // O[:, half] *= corr once PV_{j-1} has landed.  The parity test on
        // buffer (j-1)%3's barrier cannot alias: its previous phase (PV_{j-4})
        // completed before S_j was issued into buffer j%3 (in-order pipe).
        mbar_wait(bar_pvdone((j - 1) % NSB), ((j - 1) / NSB) & 1);
        __syncwarp();  // reconverge before tcgen05.ld/st (.sync.aligned)
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < HALF / 32; ++c) {
          uint32_t o[32];
          tmem_ld32(tO + lane_off + c * 32, o);
          tmem_wait_ld32(o);
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
          tmem_st32(tO + lane_off + c * 32, o);
        }
        tmem_wait_st();
      }
      tc_fence_before();
      __syncwarp();  // every lane's P store + O rescale precede the warp's arrive
      if (lane == 0) {
          if constexpr (CTAS == 2) mbar_arrive_cluster(to_leader(bar_pfull(b)));
          else mbar_arrive(bar_pfull(b));
        }
    }
    // epilogue: combine the two partial row sums, O[:, half] / l -> global
    if constexpr (NSPLIT > 1) {
      float* xl = xch + 2 * NSPLIT * 128;
      xl[hf * 128 + m] = l;
      asm volatile("bar.sync 1, %0;" ::"n"(NSM) : "memory");
      float lt = 0.f;
#pragma unroll
      for (int o = 0; o < NSPLIT; ++o) lt += xl[o * 128 + m];
      l = lt;
    }
    mbar_wait(bar_pvdone((nb - 1) % NSB), ((nb - 1) / NSB) & 1);  // PV_{nb-1} done
    __syncwarp();
    tc_fence_after();
    const float inv = valid ? 1.f / l : 0.f;
    const int64_t orow = ((int64_t)a * p.Hq + (int64_t)g * p.G + hj) * HD + hf * HALF;
#pragma unroll 1
    for (int c = 0; c < HALF / 32; ++c) {
      uint32_t o[32];
      tmem_ld32(tO + lane_off + c * 32, o);
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
  }
  tc_fence_before();
  if constexpr (CTAS == 2) cluster_sync_all();  // both CTAs done with TMEM and barriers
  else __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    if constexpr (CTAS == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512)
                   : "memory");
  }
}

// ---------------------------------------------------------------------------
// Ping-pong kernel: two 128-row query tiles (X = 0, 1: adjacent query blocks
// of one kv head) per CTA share every K/V tile.  TMEM = S_0 | S_1 | O_0 | O_1
// (128 columns each; P_X aliases the first half of S_X).  One softmax thread
// per tile row (warps 0-3 tile 0, warps 4-7 tile 1, so every SMSP runs one
// warp of each tile), and the MMA order
//     S_0(0) S_1(0) | PV_0(j) S_0(j+1) PV_1(j) S_1(j+1) | ...
// keeps one tile's MMAs in the pipe while the other tile's softmax runs, so
// the two softmax warps of an SMSP are out of phase and the exp2 (MUFU) work
// of one overlaps the TMEM load / row max / P store of the other.  K/V bytes
// per FLOP from L2 halve versus the single-tile kernel.
// ---------------------------------------------------------------------------
template <int SLOTS_ = 5>
struct SmemPP {
  static constexpr int SLOTS = SLOTS_;
  static constexpr int Q = 0;                        // two Q tiles
  static constexpr int KV = Q + 2 * TILE_BYTES;
  static constexpr int BAR = KV + SLOTS * TILE_BYTES;
  // q, full[SLOTS], empty[SLOTS], per tile: sfull, pfull, pvdone
  static constexpr int NBAR = 1 + 2 * SLOTS + 6;
  // split-row variant: [2 parity][2 tiles][2 halves][128 rows] f32 max / sum exchange
  static constexpr int XCH = BAR + NBAR * 8;
  static constexpr int XCH_BYTES = SLOTS_ < 5 ? 2 * 2 * 2 * 128 * 4 : 0;
  static constexpr int TMEM_PTR = XCH + XCH_BYTES;
  static constexpr int TOTAL = TMEM_PTR + 16;
};

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// SPLIT = 2: two softmax threads per tile row (16 softmax warps; warp
// x*8 + h*4 + q owns TMEM lane quarter q of tile x and key columns
// [64h, 64h+64) of every block), halving the per-tile S -> softmax -> PV
// latency; the two halves agree on the running max through a 64-thread named
// barrier per lane quarter, P of half h lands in TMEM columns [64h, 64h+32) of
// S, and each half rescales / stores its 64 O columns.  Needs the exchange
// area, so it runs with 4 K/V slots.
template <uint32_t POLY_MASK, int SCHED = 1, int SPLIT = 1, int SLOTS = 5>
__global__ void __launch_bounds__(32 * (8 * SPLIT + 2), 1)
attention_pp_kernel(const __grid_constant__ CUtensorMap map_q,
                    const __grid_constant__ CUtensorMap map_k,
                    const __grid_constant__ CUtensorMap map_v, const Params p) {
  using SM = SmemPP<SLOTS>;
  constexpr int TMA_WARP = 8 * SPLIT, MMA_WARP = 8 * SPLIT + 1;
  constexpr int NSLOT = SM::SLOTS;
  static_assert(SPLIT == 1 || (SPLIT == 2 && SM::XCH_BYTES > 0), "split rows need the exchange area");
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = su32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sQ = base + SM::Q, sKV = base + SM::KV;
  const uint32_t bar0 = base + SM::BAR;
  const uint32_t bar_q = bar0;
  auto bar_full = [&](int s) { return bar0 + (1 + s) * 8; };
  auto bar_empty = [&](int s) { return bar0 + (1 + NSLOT + s) * 8; };
  constexpr int B2 = 1 + 2 * NSLOT;
  auto bar_sfull = [&](int x) { return bar0 + (B2 + x) * 8; };
  auto bar_pfull = [&](int x) { return bar0 + (B2 + 2 + x) * 8; };
  auto bar_pvdone = [&](int x) { return bar0 + (B2 + 4 + x) * 8; };
  uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(gbase + SM::TMEM_PTR);
  float* xch = reinterpret_cast<float*>(gbase + SM::XCH);  // [parity][tile][half][row]

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // longest units first; unit = two adjacent query blocks of kv head g
  const int n_units = (p.n_qblocks + 1) / 2;
  const int qb0 = (n_units - 1 - (int)(blockIdx.x / p.Hkv)) * 2;
  const int g = blockIdx.x % p.Hkv;
  int maxpos = 0;
  for (int i = 0; i < 2 * p.QB; ++i) {
    const int a = qb0 * p.QB + i;
    if (a < p.A) maxpos = max(maxpos, __ldg(p.qpos + a));
  }
  maxpos = min(maxpos, p.n_ctx - 1);
  const int nb = maxpos / BLK_N + 1;

  if (threadIdx.x == 0) {
    mbar_init(bar_q, 1);
    for (int s = 0; s < NSLOT; ++s) {
      mbar_init(bar_full(s), 1);
      mbar_init(bar_empty(s), 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(bar_sfull(x), 1);
      mbar_init(bar_pfull(x), 4 * SPLIT);  // one elected arrive per softmax warp of the tile
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
      mbar_expect_tx(bar_q, 2 * TILE_BYTES);
      for (int x = 0; x < 2; ++x) {
        const int a0 = (qb0 + x) * p.QB;
        tma_load_3d(sQ + x * TILE_BYTES, &map_q, bar_q, 0, g * p.G, a0);
        tma_load_3d(sQ + x * TILE_BYTES + ATOM_BYTES, &map_q, bar_q, 64, g * p.G, a0);
      }
      int slot = 0;
      uint32_t phase = 0;
      auto load = [&](const CUtensorMap* m, int j) {
        mbar_wait(bar_empty(slot), phase ^ 1);
        const uint32_t dst = sKV + slot * TILE_BYTES;
        mbar_expect_tx(bar_full(slot), TILE_BYTES);
        tma_load_3d(dst, m, bar_full(slot), 0, g, j * BLK_N);
        tma_load_3d(dst + ATOM_BYTES, m, bar_full(slot), 64, g, j * BLK_N);
        if (++slot == NSLOT) { slot = 0; phase ^= 1; }
      };
      for (int j = 0; j < nb; ++j) {  // consumption order: K0 V0 K1 V1 ...
        load(&map_k, j);
        load(&map_v, j);
      }
    }
  } else if (warp == MMA_WARP) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t IDESC_S = idesc_bf16(false);
      constexpr uint32_t IDESC_O = idesc_bf16(true);
      mbar_wait(bar_q, 0);
      tc_fence_after();
      // K_j lives in slot (2j) % NSLOT, V_j in (2j+1) % NSLOT
      auto slot_of = [&](int i) { return i % NSLOT; };
      auto par_of = [&](int i) { return (uint32_t)((i / NSLOT) & 1); };
      auto issue_s = [&](int x, int j) {
        const int i = 2 * j, s = slot_of(i);
        if (x == 0) {
          mbar_wait(bar_full(s), par_of(i));
          tc_fence_after();
        }
        // descriptors are linear in the (16-B unit) start address: build the
        // tile's once and step them by the K-slice offset
        const uint64_t qd = sdesc(sQ + x * TILE_BYTES, 16, 1024);
        const uint64_t kd = sdesc(sKV + s * TILE_BYTES, 16, 1024);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          const uint32_t off16 = ((kk >> 2) * ATOM_BYTES + (kk & 3) * 32) >> 4;
          tc_mma(tS(x), qd + off16, kd + off16, IDESC_S, kk > 0);
        }
        if (x == 1) tc_commit(bar_empty(s));
        tc_commit(bar_sfull(x));
      };
      auto issue_pv = [&](int x, int j) {
        const int i = 2 * j + 1, s = slot_of(i);
        mbar_wait(bar_pfull(x), (uint32_t)(j & 1));
        if (x == 0) mbar_wait(bar_full(s), par_of(i));
        tc_fence_after();
        const uint64_t vd = sdesc(sKV + s * TILE_BYTES, ATOM_BYTES, 1024);
#pragma unroll
        for (int kk = 0; kk < BLK_N / 16; ++kk) {
          // P of keys [16kk, 16kk+16): bf16x2 columns 8kk (one softmax thread
          // per row) or 64*(kk/4) + 8*(kk%4) (half h stores over its own S columns)
          const uint32_t pcol = SPLIT == 1 ? kk * 8 : (kk >> 2) * 64 + (kk & 3) * 8;
          tc_mma_ts(tO(x), tS(x) + pcol, vd + (uint64_t)(kk * 2048 / 16), IDESC_O,
                    (j > 0 || kk > 0) ? 1u : 0u);
        }
        if (x == 1) tc_commit(bar_empty(s));
        tc_commit(bar_pvdone(x));
      };
      issue_s(0, 0);
      issue_s(1, 0);
      for (int j = 0; j < nb; ++j) {
        // S_x(j+1) overwrites the columns PV_x(j) reads as P: same thread,
        // in-order tcgen05.mma pipe, so it is issued right behind it
        issue_pv(0, j);
        if (j + 1 < nb) issue_s(0, j + 1);
        issue_pv(1, j);
        if (j + 1 < nb) issue_s(1, j + 1);
      }
    }
  } else {
    // ------------------------------------------------------------ softmax
    constexpr int KEYS = BLK_N / SPLIT;       // key columns per softmax thread
    const int x = warp / (4 * SPLIT);         // tile
    const int hh = SPLIT == 1 ? 0 : (warp >> 2) & 1;  // key-column half
    const int col0 = hh * KEYS;
    const int m = (warp & 3) * 32 + lane;     // TMEM lane / tile row
    const int xbar = 1 + x * 4 + (warp & 3);  // named barrier of the row's two halves
    const int qi = m / p.G, hj = m % p.G;
    const int a = (qb0 + x) * p.QB + qi;
    const bool valid = a < p.A;
    const int pos = valid ? min(__ldg(p.qpos + a), p.n_ctx - 1) : maxpos;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    float m_used = -INFINITY, l = 0.f;
    uint32_t r[KEYS];
    for (int j = 0; j < nb; ++j) {
      mbar_wait(bar_sfull(x), (uint32_t)(j & 1));
      __syncwarp();
      tc_fence_after();
      if constexpr (SCHED == 4) {  // timing probe (wrong values): MMA + TMA pipeline alone
        l = 1.f;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar_pfull(x));
        continue;
      }
#pragma unroll
      for (int c = 0; c < KEYS / 32; ++c) tmem_ld32(tS(x) + lane_off + col0 + c * 32, r + c * 32);
#pragma unroll
      for (int c = 0; c < KEYS / 32; ++c) tmem_wait_ld32(r + c * 32);
      const int kbase = j * BLK_N + col0;
      const bool need_mask = kbase + KEYS - 1 > pos;
      if (need_mask) {
#pragma unroll
        for (int c = 0; c < KEYS; ++c)
          if (kbase + c > pos) r[c] = __float_as_uint(-INFINITY);
      }
      float mq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int c = 0; c < KEYS; c += 8) {
#pragma unroll
        for (int t = 0; t < 4; ++t)
          mq[t] = max3f(mq[t], __uint_as_float(r[c + 2 * t]), __uint_as_float(r[c + 2 * t + 1]));
      }
      float mx = max3f(mq[0], mq[1], fmaxf(mq[2], mq[3])) * p.scale_log2;
      if constexpr (SPLIT == 2) {
        // both halves of the row must use the same running max: exchange the
        // block maxima (double buffered by block parity, so a fast half never
        // overwrites a value its partner has not read yet)
        float* xb = xch + (((j & 1) * 2 + x) * 2) * 128;
        xb[hh * 128 + m] = mx;
        named_bar_sync(xbar, 64);
        mx = fmaxf(mx, xb[(hh ^ 1) * 128 + m]);  // symmetric: both halves get the same value
      }
      const float m_new = fmaxf(m_used, mx);
      const bool grow = m_new > m_used + p.lazy_thresh;
      const bool any_grow = __any_sync(0xffffffffu, grow);
      const float corr = grow ? ex2(m_used - m_new) : 1.f;  // 0 when m_used = -inf
      if (grow) m_used = m_new;
      const uint64_t sc2 = pk2(p.scale_log2, p.scale_log2);
      const uint64_t nm2 = pk2(-m_used, -m_used);
      uint64_t acc2[2] = {pk2(0.f, 0.f), pk2(0.f, 0.f)};
      // P_j (bf16x2) -> TMEM columns [0, 64) of S_x, 32 keys per store
      if constexpr (SCHED == 0 && SPLIT == 1) {
        auto chunk = [&](auto cc) {
          constexpr int c = decltype(cc)::value;
          uint32_t pk[16];
          if (need_mask)
            softmax_chunks<32, 0u>(r + c * 32, sc2, nm2, acc2, pk);
          else
            softmax_chunks<32, (POLY_MASK >> (4 * c)) & 0xFu>(r + c * 32, sc2, nm2, acc2, pk);
          tmem_st16(tS(x) + lane_off + c * 16, pk);
        };
        chunk(std::integral_constant<int, 0>{});
        chunk(std::integral_constant<int, 1>{});
        chunk(std::integral_constant<int, 2>{});
        chunk(std::integral_constant<int, 3>{});
      } else {
        // phased, per half block (64 keys): the FFMA2 arguments, then the exp2
        // run back to back (MUFU / polynomial), then packing + row sums + TMEM
        // stores, so one warp keeps the MUFU pipe fed without per-chunk chains
#pragma unroll
        for (int hb = 0; hb < KEYS / 64; ++hb) {
          uint32_t* rh = r + hb * 64;
#pragma unroll
          for (int c = 0; c < 64; c += 2) {
            const uint64_t a2 = ffma2(pk2(__uint_as_float(rh[c]), __uint_as_float(rh[c + 1])), sc2, nm2);
            float a, b;
            upk2(a2, a, b);
            rh[c] = __float_as_uint(a);
            rh[c + 1] = __float_as_uint(b);
          }
          if (SCHED == 3) {  // timing probe (wrong values): exp2 replaced by an FMUL
#pragma unroll
            for (int c = 0; c < 64; ++c) rh[c] = __float_as_uint(__uint_as_float(rh[c]) * 0.5f);
          } else if (need_mask) {
#pragma unroll
            for (int c = 0; c < 64; ++c) rh[c] = __float_as_uint(ex2(__uint_as_float(rh[c])));
          } else {
#pragma unroll
            for (int c = 0; c < 64; c += 2) {
              if ((POLY_MASK >> ((col0 + hb * 64 + c) / 8)) & 1) {
                uint32_t o0, o1;
                exp2_poly2(pk2(__uint_as_float(rh[c]), __uint_as_float(rh[c + 1])), o0, o1);
                rh[c] = o0;
                rh[c + 1] = o1;
              } else {
                rh[c] = __float_as_uint(ex2(__uint_as_float(rh[c])));
                rh[c + 1] = __float_as_uint(ex2(__uint_as_float(rh[c + 1])));
              }
            }
          }
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            uint32_t pk[16];
#pragma unroll
            for (int t = 0; t < 16; ++t) {
              const uint32_t e0 = rh[c * 32 + 2 * t], e1 = rh[c * 32 + 2 * t + 1];
              acc2[t & 1] = fadd2(acc2[t & 1], (uint64_t)e0 | ((uint64_t)e1 << 32));
              pk[t] = pack_bf16(__uint_as_float(e0), __uint_as_float(e1));
            }
            tmem_st16(tS(x) + lane_off + col0 + (hb * 2 + c) * 16, pk);
          }
        }
      }
      {
        float s0, s1, s2, s3;
        upk2(acc2[0], s0, s1);
        upk2(acc2[1], s2, s3);
        l = l * corr + ((s0 + s1) + (s2 + s3));
      }
      tmem_wait_st();
      if (any_grow && j > 0) {
        // O_x *= corr once PV_x(j-1) has landed (warp-uniform branch)
        mbar_wait(bar_pvdone(x), (uint32_t)((j - 1) & 1));
        __syncwarp();
        tc_fence_after();
#pragma unroll 1
        for (int c = 0; c < HD / 32 / SPLIT; ++c) {
          const uint32_t oc = hh * (HD / SPLIT) + c * 32;
          uint32_t o[32];
          tmem_ld32(tO(x) + lane_off + oc, o);
          tmem_wait_ld32(o);
#pragma unroll
          for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * corr);
          tmem_st32(tO(x) + lane_off + oc, o);
        }
        tmem_wait_st();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_pfull(x));
    }
    mbar_wait(bar_pvdone(x), (uint32_t)((nb - 1) & 1));
    __syncwarp();
    tc_fence_after();
    if constexpr (SPLIT == 2) {
      float* xb = xch + (((nb & 1) * 2 + x) * 2) * 128;
      xb[hh * 128 + m] = l;
      named_bar_sync(xbar, 64);
      l = l + xb[(hh ^ 1) * 128 + m];  // commutative: both halves agree
    }
    const float inv = valid ? 1.f / l : 0.f;
    const int64_t orow = ((int64_t)a * p.Hq + (int64_t)g * p.G + hj) * HD;
#pragma unroll 1
    for (int cc = 0; cc < HD / 32 / SPLIT; ++cc) {
      const int c = hh * (HD / 32 / SPLIT) + cc;
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

}  // namespace tc

bool tc_enabled() { return true; }

size_t attention_tc_workspace(int64_t, int64_t, int64_t, int64_t, int64_t) { return 0; }

int attention_tc(const void* q, const int32_t* q_pos, int64_t A, int64_t Hq, const void* k_cache,
                 const void* v_cache, int64_t n_ctx, int64_t Hkv, int64_t D,
                 int64_t cache_row_stride, double scale, void* out, int out_dtype,
                 void* workspace, size_t workspace_bytes, cudaStream_t st) {
  using namespace tc;
  (void)workspace;
  (void)workspace_bytes;
  if (D != HD) return fail(CT_ERR_UNSUPPORTED, "tcgen05 attention needs head_dim 128");
  const int64_t G = Hq / Hkv;
  if (G < 1 || TILE_M % G) return fail(CT_ERR_UNSUPPORTED, "GQA group %lld must divide 128", (long long)G);
  if (((uintptr_t)q | (uintptr_t)k_cache | (uintptr_t)v_cache) & 15)
    return fail(CT_ERR_PARAM, "tensors must be 16-byte aligned");
  if ((cache_row_stride * 2) % 16) return fail(CT_ERR_PARAM, "cache row stride alignment");
  CUtensorMap mq, mk, mv;
  int rc;
  if ((rc = make_map(&mq, q, (uint64_t)Hq, (uint64_t)A, HD * 2, (uint64_t)Hq * HD * 2,
                     (uint32_t)G, (uint32_t)(TILE_M / G))))
    return rc;
  const int kbox = (getenv("CT_TC_CTAS") && atoi(getenv("CT_TC_CTAS")) == 2) ? BLK_N / 2 : BLK_N;
  if ((rc = make_map(&mk, k_cache, (uint64_t)Hkv, (uint64_t)n_ctx, HD * 2,
                     (uint64_t)cache_row_stride * 2, 1, (uint32_t)kbox)))
    return rc;
  if ((rc = make_map(&mv, v_cache, (uint64_t)Hkv, (uint64_t)n_ctx, HD * 2,
                     (uint64_t)cache_row_stride * 2, 1, BLK_N)))
    return rc;
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
  prm.lazy_thresh = LAZY_THRESH;
  if (const char* e = getenv("CT_TC_LAZY")) prm.lazy_thresh = (float)atof(e);
  // Single-CTA tiles by default.  CT_TC_CTAS=2 selects the CTA-pair kernel
  // (cta_group::2, MMA M = 256, half of every K/V tile per SM): correct and it
  // halves L2->SM traffic, but measured 40 % slower (its 2-SM TMA pipeline
  // starves the MMA; profiles/round1_attention_variants.md).  CT_TC_EXPT /
  // CT_TC_POLY are profiling aids.
  int ctas = 1;
  if (const char* e = getenv("CT_TC_CTAS")) ctas = atoi(e) == 2 ? 2 : 1;
  // exp2 on MUFU only: with the phased softmax the FMA-pipe polynomial no
  // longer pays (profiles/round1_attention_variants.md); CT_TC_POLY selects it
  uint32_t poly = 0;
  if (const char* e = getenv("CT_TC_POLY")) poly = (uint32_t)strtoul(e, nullptr, 0);
  int expt = 0;
  if (const char* e = getenv("CT_TC_EXPT")) expt = atoi(e);
  using KernFn = void (*)(CUtensorMap, CUtensorMap, CUtensorMap, Params);
  KernFn kern;
  int pp = 1;
  if (const char* e = getenv("CT_TC_PP")) pp = atoi(e);
  if (pp && ctas == 1 && expt == 0) {
    int sched = 1;
    if (const char* e = getenv("CT_TC_SCHED")) sched = atoi(e);
    KernFn kp = sched == 0 ? (poly == 0x4444 ? attention_pp_kernel<0x4444u, 0> : attention_pp_kernel<0u, 0>)
              : sched == 3 ? attention_pp_kernel<0u, 3>
              : sched == 4 ? attention_pp_kernel<0u, 4>
              : poly == 0x3333 ? attention_pp_kernel<0x3333u>
              : poly == 0x7777 ? attention_pp_kernel<0x7777u>
              : poly == 0xFFFF ? attention_pp_kernel<0xFFFFu>
              : poly == 0x4444 ? attention_pp_kernel<0x4444u>
              : poly == 0x0202 ? attention_pp_kernel<0x0202u>
              : poly == 0x5555 ? attention_pp_kernel<0x5555u>
              : poly == 0x1111 ? attention_pp_kernel<0x1111u>
              : poly == 0x2222 ? attention_pp_kernel<0x2222u> : attention_pp_kernel<0u>;
    int split = 1;
    if (const char* e = getenv("CT_TC_SPLIT")) split = atoi(e) == 2 ? 2 : 1;
    // split rows (neutral on the selective shape; the FMA-pipe polynomial in
    // the key half of one warp set measured much slower,
    // profiles/round1_attention_variants.md)
    if (split == 2) kp = attention_pp_kernel<0u, 1, 2, 4>;
    const size_t smem_pp = (split == 2 ? SmemPP<4>::TOTAL : SmemPP<5>::TOTAL) + 1024;
    CT_CUDA(cudaFuncSetAttribute(kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_pp));
    const unsigned grid_pp = (unsigned)(((prm.n_qblocks + 1) / 2) * Hkv);
    kp<<<grid_pp, 32 * (8 * split + 2), smem_pp, st>>>(mq, mk, mv, prm);
    return check_launch("attention_pp_kernel");
  }
  if (ctas == 2)
    kern = expt == 1 ? attention_tc_kernel<2, 0, 1, 2> : expt == 2 ? attention_tc_kernel<2, 0, 2, 2>
         : expt == 3 ? attention_tc_kernel<2, 0, 3, 2> : expt == 4 ? attention_tc_kernel<2, 0, 4, 2>
         : poly == 0x22 ? attention_tc_kernel<2, 0x22, 0, 2> : attention_tc_kernel<2, 0, 0, 2>;
  else
    kern = expt == 1 ? attention_tc_kernel<2, 0, 1, 1> : expt == 2 ? attention_tc_kernel<2, 0, 2, 1>
         : expt == 4 ? attention_tc_kernel<2, 0, 4, 1>
         : poly == 0x22 ? attention_tc_kernel<2, 0x22, 0, 1> : attention_tc_kernel<2, 0, 0, 1>;
  const size_t smem = (ctas == 2 ? Smem<2>::TOTAL : Smem<1>::TOTAL) + 1024;
  const int threads = 32 * (4 * 2 + 2);
  CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int units = (prm.n_qblocks + ctas - 1) / ctas;
  const unsigned grid = (unsigned)(units * Hkv * ctas);
  if (ctas == 1) {
    kern<<<grid, threads, smem, st>>>(mq, mk, mv, prm);
  } else {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CT_CUDA(cudaLaunchKernelEx(&cfg, kern, mq, mk, mv, prm));
  }
  return check_launch("attention_tc_kernel");
}

}  // namespace ct
