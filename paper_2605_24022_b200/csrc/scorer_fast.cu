// Fast scorer: single-precision four-step FFT energy kernel + certified top-k
// boundary.  Same quantity as ct/spectral.py:69-79 / :149-159 (rfft along the
// token axis, keep bins min(k, N-k) < c, irfft, per-token row norms, 0.5 K +
// 0.5 V, sequential layer mean), computed for N = 2048 with float32 FFTs, and
// a selection step that proves the top-k set of the aggregate score equals
// the float64 one (ct/spectral.py:162-184):
//
//   1. fs_energy_split_kernel (default band, bf16; below) / fs_energy_kernel
//      (other bands, f32 or unaligned rows): two lanes packed per complex signal (the mask is
//      Hermitian, so lowpass(a + ib) = lowpass(a) + i lowpass(b)); the 2048
//      tokens are n = n2 + 64 n1.  Step 1: 32-point DFT over n1 in registers
//      (radix-4/2 DIF, compile-time twiddles) and the W_2048^(n2 k1) twiddle;
//      exchange 1 through shared memory; step 2: per k1 a 64-point DFT over
//      n2, the band mask, the 64-point inverse (the same stages reversed, no
//      reordering), the inverse twiddle; exchange 2; step 3: 32-point inverse
//      over k1 -> tokens n2' + 64 n1', |y|^2 accumulated per token in
//      registers over the CTA's signals.  Two shared-memory exchanges per
//      signal (XOR-swizzled, at most 2 lanes per 8-byte bank slot), K/V read
//      once with sector-complete 32-byte row pieces.
//   2. fs_combine: per token and layer 0.5 sqrt(EK) + 0.5 sqrt(EV) in f64,
//      sequential layer sum / L.
//   3. desc order (scorer.cu), then fs_window: the aggregate scores carry a
//      relative error bound g (calibrated); the k-th / (k+1)-th
//      boundary is certified when a_k (1 - g) > a_{k+1} (1 + g); otherwise
//      every token whose score lies in [a_{k+1}(1-g)/(1+g), a_k(1+g)/(1-g)]
//      is re-scored exactly (fs_rescore: float64 direct low-pass projection
//      y_i = sum_n p[(i - n) mod N] x_n over all layers, lanes and both
//      tensors) and the window is re-ordered by (exact score desc, index asc)
//      (fs_fixup).  Tokens outside the window provably keep their side of the
//      boundary, so order[0..k) is the exact top-k set.  Windows wider than
//      FS_WMAX tokens are reported; the host re-scores those chunks with the
//      exact (float64) scorer.
#include "common.cuh"

namespace ct {
namespace fs {

constexpr int N = 2048;
constexpr int THREADS = 256;
constexpr int SIG_PER_BATCH = 8;
constexpr int BATCHES = 8;                       // signals per CTA = 64 (128 lanes)
constexpr int SIG_PER_CTA = SIG_PER_BATCH * BATCHES;
constexpr int WMAX = 64;                         // window tokens re-scored per chunk

__device__ constexpr float kCos64[64] = {
#include "scorer_fast_cos64.inc"
};
__device__ constexpr float kSin64[64] = {
#include "scorer_fast_sin64.inc"
};

// complex f32 as float2: adds / subs / twiddle products are packed FADD2 /
// FMUL2 / FFMA2 (one issue slot per complex add, two per complex product)
using cf = float2;
__device__ __forceinline__ cf operator+(cf a, cf b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ cf operator-(cf a, cf b) {
  return __fadd2_rn(a, make_float2(-b.x, -b.y));
}
// a * (i * SG), SG = +-1
template <int SG>
__device__ __forceinline__ cf mul_i(cf a) {
  return SG > 0 ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x);
}
// a * exp(SG * 2 pi i * m / 64) with exact trivial factors
template <int SG, int M>
__device__ __forceinline__ cf tw64(cf a) {
  constexpr int m = ((M % 64) + 64) % 64;
  if constexpr (m == 0) {
    return a;
  } else if constexpr (m == 16) {
    return mul_i<SG>(a);
  } else if constexpr (m == 32) {
    return make_float2(-a.x, -a.y);
  } else if constexpr (m == 48) {
    return mul_i<-SG>(a);
  } else {
    // (x c - y s, x s + y c) = x (c, s) + y (-s, c)
    const float c = kCos64[m], s = SG * kSin64[m];
    const cf r = __fmul2_rn(make_float2(a.x, a.x), make_float2(c, s));
    return __ffma2_rn(make_float2(a.y, a.y), make_float2(-s, c), r);
  }
}
__device__ __forceinline__ cf cmul(cf a, cf w) {
  const cf r = __fmul2_rn(make_float2(a.x, a.x), w);
  return __ffma2_rn(make_float2(a.y, a.y), make_float2(-w.y, w.x), r);
}
__device__ __forceinline__ cf cmulc(cf a, cf w) {  // a * conj(w)
  const cf r = __fmul2_rn(make_float2(a.x, a.x), make_float2(w.x, -w.y));
  return __ffma2_rn(make_float2(a.y, a.y), make_float2(w.y, w.x), r);
}

// Radix-4 DIF stage of span SPAN over v[M] (SG = -1: forward DFT kernel).
template <int M, int SPAN, int SG>
__device__ __forceinline__ void dif_stage(cf (&v)[M]) {
  constexpr int Q = SPAN / 4, F = 64 / SPAN;
#pragma unroll
  for (int g = 0; g < M; g += SPAN) {
#pragma unroll
    for (int j = 0; j < Q; ++j) {
      const cf a = v[g + j], b = v[g + j + Q], c = v[g + j + 2 * Q], d = v[g + j + 3 * Q];
      const cf t0 = a + c, t1 = a - c, t2 = b + d, t3 = mul_i<SG>(b - d);
      v[g + j] = t0 + t2;
      v[g + j + Q] = t1 + t3;
      v[g + j + 2 * Q] = t0 - t2;
      v[g + j + 3 * Q] = t1 - t3;
    }
  }
}
// twiddles of a DIF stage (applied after its butterflies): position j + rQ
// of each group times W_SPAN^(r j)
template <int M, int SPAN, int SG, int J = 0>
__device__ __forceinline__ void dif_twiddle(cf (&v)[M]) {
  constexpr int Q = SPAN / 4, F = 64 / SPAN;
  if constexpr (J < Q) {
#pragma unroll
    for (int g = 0; g < M; g += SPAN) {
      v[g + J + Q] = tw64<SG, F * J>(v[g + J + Q]);
      v[g + J + 2 * Q] = tw64<SG, F * 2 * J>(v[g + J + 2 * Q]);
      v[g + J + 3 * Q] = tw64<SG, F * 3 * J>(v[g + J + 3 * Q]);
    }
    dif_twiddle<M, SPAN, SG, J + 1>(v);
  }
}
// inverse of dif_stage + dif_twiddle (conjugate twiddles first, then the
// transposed butterfly); unnormalised
template <int M, int SPAN, int SG, int J = 0>
__device__ __forceinline__ void dit_twiddle(cf (&v)[M]) {
  constexpr int Q = SPAN / 4, F = 64 / SPAN;
  if constexpr (J < Q) {
#pragma unroll
    for (int g = 0; g < M; g += SPAN) {
      v[g + J + Q] = tw64<SG, F * J>(v[g + J + Q]);
      v[g + J + 2 * Q] = tw64<SG, F * 2 * J>(v[g + J + 2 * Q]);
      v[g + J + 3 * Q] = tw64<SG, F * 3 * J>(v[g + J + 3 * Q]);
    }
    dit_twiddle<M, SPAN, SG, J + 1>(v);
  }
}
template <int M, int SPAN, int SG>
__device__ __forceinline__ void dit_stage(cf (&v)[M]) {
  constexpr int Q = SPAN / 4;
#pragma unroll
  for (int g = 0; g < M; g += SPAN) {
#pragma unroll
    for (int j = 0; j < Q; ++j) {
      const cf y0 = v[g + j], y1 = v[g + j + Q], y2 = v[g + j + 2 * Q], y3 = v[g + j + 3 * Q];
      const cf t0 = y0 + y2, t2 = y0 - y2, t1 = y1 + y3, t3 = mul_i<SG>(y1 - y3);
      v[g + j] = t0 + t1;
      v[g + j + 2 * Q] = t0 - t1;
      v[g + j + Q] = t2 + t3;
      v[g + j + 3 * Q] = t2 - t3;
    }
  }
}
template <int M>
__device__ __forceinline__ void radix2(cf (&v)[M]) {
#pragma unroll
  for (int g = 0; g < M; g += 2) {
    const cf a = v[g], b = v[g + 1];
    v[g] = a + b;
    v[g + 1] = a - b;
  }
}

// Forward DFT (natural order in, digit-reversed out) and its exact reverse
// (digit-reversed in, natural out, conjugate kernel): M = 32 (4, 4, 2), 64 (4, 4, 4).
template <int M>
__device__ __forceinline__ void fwd(cf (&v)[M]) {
  dif_stage<M, M, -1>(v);
  dif_twiddle<M, M, -1>(v);
  dif_stage<M, M / 4, -1>(v);
  dif_twiddle<M, M / 4, -1>(v);
  if constexpr (M == 64) {
    dif_stage<M, 4, -1>(v);
  } else {
    radix2<M>(v);
  }
}
template <int M>
__device__ __forceinline__ void inv(cf (&v)[M]) {
  if constexpr (M == 64) {
    dit_stage<M, 4, 1>(v);
  } else {
    radix2<M>(v);
  }
  dit_twiddle<M, M / 4, 1>(v);
  dit_stage<M, M / 4, 1>(v);
  dit_twiddle<M, M, 1>(v);
  dit_stage<M, M, 1>(v);
}
// frequency held at output position p of fwd<M> (digit reversal)
template <int M>
__host__ __device__ constexpr int digrev(int p) {
  if (M == 64) return ((p & 3) << 4) | (p & 12) | (p >> 4);
  // 32: digits (base 4, base 4, base 2) of the DIF order
  return ((p & 1) << 4) | (((p >> 1) & 3) << 2) | (p >> 3);
}

// exchange buffer index (8-byte units): [s][k1][n2 ^ swz(s, k1)].  An 8-byte
// access is served per half-warp (16 lanes x 8 B = one wavefront); in every
// exchange pattern a half-warp holds 8 signal slots s and two k1 or two n2
// values, and swz = 2s ^ (k1 & 1) maps them onto 16 distinct 8-byte slots.
__device__ __forceinline__ int xidx(int s, int k1, int n2) {
  return ((s * 32 + k1) << 6) + (n2 ^ ((s << 1) ^ (k1 & 1)));
}

template <typename IN>
__device__ __forceinline__ cf load_pair(const IN* p);
template <>
__device__ __forceinline__ cf load_pair<__nv_bfloat16>(const __nv_bfloat16* p) {
  const uint32_t u = __ldg(reinterpret_cast<const unsigned int*>(p));
  return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
}
template <>
__device__ __forceinline__ cf load_pair<float>(const float* p) {
  return __ldg(reinterpret_cast<const float2*>(p));
}

__device__ __forceinline__ void cp_async16(const void* dst_smem, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst_smem)),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ cf unpack_bf16x2(uint32_t u) {
  return make_float2(__uint_as_float(u << 16), __uint_as_float(u & 0xffff0000u));
}
// bf16 inputs with 16-byte aligned rows: a batch's 16 lanes x 2048 tokens
// (32 B per token, 64 KiB) are staged in shared memory by cp.async one batch
// ahead, so step 1 reads shared memory while the next batch is in flight.
constexpr size_t STAGE_BYTES = (size_t)N * SIG_PER_BATCH * 4;

// grid: x = lane group (SIG_PER_CTA signals), y = tensor (0 K, 1 V), z = c*L + l.
// partial[((c*L + l)*2 + tensor)*G + group][N] f32 (unnormalised |y|^2, x N^2)
template <typename IN, bool STAGE, bool LB>
__global__ void __launch_bounds__(THREADS, 1)
fs_energy_kernel(const IN* __restrict__ keys, const IN* __restrict__ values, int L,
                 int64_t ld_token, int64_t ld_layer, int64_t ld_chunk, int cutoff, int high,
                 const float2* __restrict__ tw, int groups, float* __restrict__ partial) {
  static_assert(!STAGE || sizeof(IN) == 2, "staging is for bf16 rows");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cf* xb = reinterpret_cast<cf*>(smem_raw);                  // [8][32][64]
  cf* T = xb + SIG_PER_BATCH * 32 * 64;                       // W_2048^m, m < 2048
  uint32_t* stg = reinterpret_cast<uint32_t*>(T + N);         // [N][8] bf16x2 (STAGE)
  const int t = threadIdx.x, s = t & 7, q = t >> 3;
  const int tensor = blockIdx.y, group = blockIdx.x;
  const int c = blockIdx.z / L, l = blockIdx.z % L;
  for (int i = t; i < N; i += THREADS) T[i] = tw[i];
  const IN* base = (tensor ? values : keys) + (int64_t)c * ld_chunk + (int64_t)l * ld_layer +
                   (int64_t)group * SIG_PER_CTA * 2;
  // energies of tokens q + 32 (s >> 2) + 64 (8 (s & 3) + i), i < 8: the
  // batch's |y|^2 of the 8 signal slots are reduce-scattered over the 8 lanes
  // of one q, so each lane keeps 8 token sums instead of 64
  float acc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = 0.f;
  // batch b's 16 lanes of every token: thread t moves 16-byte halves (t & 1)
  // of token rows t/2 + 128 i (sector-complete 32-byte row pieces per pair)
  auto prefetch = [&](int b) {
    const IN* src = base + b * SIG_PER_BATCH * 2 + (t & 1) * 8 + (int64_t)(t >> 1) * ld_token;
    uint32_t* dst = stg + (t >> 1) * SIG_PER_BATCH + (t & 1) * 4;
    const int64_t step = (int64_t)(THREADS / 2) * ld_token;
#pragma unroll 1
    for (int i = 0; i < N / (THREADS / 2); ++i) {
      cp_async16(dst, src);
      src += step;
      dst += (THREADS / 2) * SIG_PER_BATCH;
    }
    cp_async_commit();
  };
  if constexpr (STAGE) prefetch(0);
  __syncthreads();

#pragma unroll 1
  for (int b = 0; b < BATCHES; ++b) {
    const IN* sig = base + (b * SIG_PER_BATCH + s) * 2;
    if constexpr (STAGE) {
      cp_async_wait_all();
      __syncthreads();
    }
    // ---- step 1: 32-point DFT over n1 of tokens n2 + 64 n1, twiddle, exchange
#pragma unroll
    for (int jb = 0; jb < 2; ++jb) {
      const int n2 = q + 32 * jb;
      cf v[32];
#pragma unroll
      for (int n1 = 0; n1 < 32; ++n1) {
        if constexpr (STAGE)
          v[n1] = unpack_bf16x2(stg[(n2 + 64 * n1) * SIG_PER_BATCH + s]);
        else
          v[n1] = load_pair<IN>(sig + (int64_t)(n2 + 64 * n1) * ld_token);
      }
      fwd<32>(v);
#pragma unroll
      for (int p = 0; p < 32; ++p) {
        const int k1 = digrev<32>(p);
        xb[xidx(s, k1, n2)] = cmul(v[p], T[(n2 * k1) & (N - 1)]);
      }
    }
    __syncthreads();
    // every thread is past its staged reads: the next batch streams in
    // behind steps 2 and 3
    if constexpr (STAGE) {
      if (b + 1 < BATCHES) prefetch(b + 1);
    }
    // ---- step 2: per k1 = q: 64-point DFT over n2, band mask, inverse, twiddle
    {
      const int k1 = q;
      cf u[64];
#pragma unroll
      for (int n2 = 0; n2 < 64; ++n2) u[n2] = xb[xidx(s, k1, n2)];
      if constexpr (LB) {
        // default band (low, cutoff N/4): the last forward radix-4 stage
        // holds the top digit of k2 at position p & 3, and digits 1 and 2
        // (k2 in [16, 48)) are always cut, so that stage, the mask and the
        // first inverse stage fuse into 10 complex adds per group instead
        // of 16 -- the same operations on the surviving values as the
        // generic path below (bitwise the same energies)
        dif_stage<64, 64, -1>(u);
        dif_twiddle<64, 64, -1>(u);
        dif_stage<64, 16, -1>(u);
        dif_twiddle<64, 16, -1>(u);
#pragma unroll
        for (int g = 0; g < 64; g += 4) {
          const cf a = u[g], b = u[g + 1], c = u[g + 2], d = u[g + 3];
          const cf t0 = a + c, t1 = a - c, t2 = b + d;
          const cf x0 = t0 + t2;
          cf x3 = t1 - mul_i<-1>(b - d);
          if (g == 0 && k1 == 0) x3 = make_float2(0.f, 0.f);  // k = 3N/4 is cut
          const cf t3 = mul_i<1>(make_float2(0.f, 0.f) - x3);
          u[g] = x0 + x3;
          u[g + 2] = x0 - x3;
          u[g + 1] = x0 + t3;
          u[g + 3] = x0 - t3;
        }
        dit_twiddle<64, 16, 1>(u);
        dit_stage<64, 16, 1>(u);
        dit_twiddle<64, 64, 1>(u);
        dit_stage<64, 64, 1>(u);
      } else {
        fwd<64>(u);
#pragma unroll
        for (int p = 0; p < 64; ++p) {
          const int k = k1 + 32 * digrev<64>(p);
          const int kk = min(k, N - k);
          const bool keep = high ? kk >= cutoff : kk < cutoff;
          if (!keep) u[p] = make_float2(0.f, 0.f);
        }
        inv<64>(u);
      }
      // this thread's row of the buffer is read and written by it alone
#pragma unroll
      for (int n2 = 0; n2 < 64; ++n2) xb[xidx(s, k1, n2)] = cmulc(u[n2], T[(n2 * k1) & (N - 1)]);
    }
    __syncthreads();
    // ---- step 3: 32-point inverse over k1 -> tokens n2' + 64 n1', energies
    float e[64];
#pragma unroll
    for (int jb = 0; jb < 2; ++jb) {
      const int n2 = q + 32 * jb;
      cf w[32];
#pragma unroll
      for (int p = 0; p < 32; ++p) w[p] = xb[xidx(s, digrev<32>(p), n2)];
      inv<32>(w);
#pragma unroll
      for (int n1 = 0; n1 < 32; ++n1) e[32 * jb + n1] = fmaf(w[n1].x, w[n1].x, w[n1].y * w[n1].y);
    }
    __syncthreads();
    // reduce-scatter over s (xor 4, 2, 1): lane s ends with slots [8s, 8s + 8)
    {
      const bool b2 = s & 4, b1 = s & 2, b0 = s & 1;
      float f[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float send = b2 ? e[i] : e[32 + i];
        f[i] = (b2 ? e[32 + i] : e[i]) + __shfl_xor_sync(0xffffffffu, send, 4);
      }
      float g2[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float send = b1 ? f[i] : f[16 + i];
        g2[i] = (b1 ? f[16 + i] : f[i]) + __shfl_xor_sync(0xffffffffu, send, 2);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float send = b0 ? g2[i] : g2[8 + i];
        acc[i] += (b0 ? g2[8 + i] : g2[i]) + __shfl_xor_sync(0xffffffffu, send, 1);
      }
    }
  }
  float* out = partial + ((((int64_t)c * L + l) * 2 + tensor) * groups + group) * N;
#pragma unroll
  for (int i = 0; i < 8; ++i) out[q + 32 * (s >> 2) + 64 * (8 * (s & 3) + i)] = acc[i];
}

// ---------------------------------------------------------------------------
// Default band (low, cutoff N/4), bf16 rows, 16-byte aligned: the same
// four-step transform with 512 threads (16 warps, <= 128 registers) instead
// of 256 at 255 registers -- twice the warps per SM to hide the FMA / shared
// memory latencies of the register-resident FFT.  Step 1 and step 3 do one
// 32-point column per thread.  Step 2's 64-point row (k1) is split over a
// lane pair h = 0, 1 (lanes t, t ^ 8): lane h transforms the samples
// u[2m + h] (radix-2 decimation in time), so
//   X[k] = D0[k] + W64^k D1[k],   X[k + 32] = D0[k] - W64^k D1[k].
// The band keeps k2 < 16 (lane 0) and k2 > 48 (lane 1); everything between
// is cut, so each lane completes only its 16 surviving bins after one
// 16-value shuffle exchange, and the inverse split (D0' = X[k] + X[k+32],
// D1' = W64^-k (X[k] - X[k+32])) needs one more.  Lane 1 works on
// frequency-shifted copies so both lanes run identical code: its input is
// multiplied by (-1)^m (its DFT comes out shifted by 16), it holds
// Z = W64^-(k+48) X[k+48], and its inverse output carries a (-1)^m sign --
// a sign common to all rows of a column n2, hence to all tokens that step 3
// builds from it, so every |y|^2 is unchanged.  Per-lane twiddles come
// from two 2 x 16 shared tables.
// ---------------------------------------------------------------------------
__host__ __device__ constexpr int posof32(int f) {
  int p = 0;
  for (int i = 0; i < 32; ++i)
    if (digrev<32>(i) == f) p = i;
  return p;
}
__device__ __forceinline__ cf shfl_xor_cf(cf a, int m) {
  return make_float2(__shfl_xor_sync(0xffffffffu, a.x, m), __shfl_xor_sync(0xffffffffu, a.y, m));
}
// SIG signal slots per batch, 64 SIG threads: SIG = 8 -> one 512-thread CTA
// per SM (the product), SIG = 4 -> two 256-thread CTAs per SM (measured slower)
template <int SIG>
struct Split {
  static constexpr int THREADS = 64 * SIG;
  static constexpr int BATCHES = SIG_PER_CTA / SIG;
  static constexpr int LOG = SIG == 8 ? 3 : 2;
  static constexpr size_t STAGE = (size_t)N * SIG * 4;
  // smem: xb [SIG][32][64] cf | T [N] cf | twA [2][16] | twB [2][16] | stage
  static constexpr size_t SMEM = (size_t)SIG * 32 * 64 * sizeof(cf) + N * sizeof(cf) +
                                 64 * sizeof(cf) + STAGE;
  // exchange index: every 16-lane access pattern (steps 1/3: SIG slots x
  // 16/SIG consecutive n2; step 2: SIG slots x h x two k1) hits 16 distinct
  // 8-byte slots
  static __device__ __forceinline__ int xi(int s, int k1, int n2) {
    const int swz = SIG == 8 ? ((s << 1) ^ (k1 & 1)) : ((s << 2) ^ ((k1 & 1) << 1));
    return ((s * 32 + k1) << 6) + (n2 ^ swz);
  }
};

template <int SIG>
__global__ void __launch_bounds__(64 * SIG, 8 / SIG)
fs_energy_split_kernel(const __nv_bfloat16* __restrict__ keys,
                       const __nv_bfloat16* __restrict__ values, int L, int64_t ld_token,
                       int64_t ld_layer, int64_t ld_chunk, const float2* __restrict__ tw,
                       int groups, float* __restrict__ partial) {
  using S = Split<SIG>;
  constexpr int TH = S::THREADS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cf* xb = reinterpret_cast<cf*>(smem_raw);                  // [SIG][32][64]
  cf* T = xb + SIG * 32 * 64;                                 // W_2048^m
  cf* twA = T + N;                                            // [h][kk]
  cf* twB = twA + 32;
  uint32_t* stg = reinterpret_cast<uint32_t*>(twB + 32);      // [N][SIG] bf16x2
  const int t = threadIdx.x, s = t & (SIG - 1), q = t >> S::LOG;  // q < 64
  const int tensor = blockIdx.y, group = blockIdx.x;
  const int c = blockIdx.z / L, l = blockIdx.z % L;
  for (int i = t; i < N; i += TH) T[i] = tw[i];
  if (t < 16) {
    // forward combine: lane 0 W64^kk, lane 1 W64^-(kk+48); inverse send:
    // lane 0 W64^-kk, lane 1 W64^(kk+48)  (W64^m = W2048^(32 m))
    twA[t] = tw[32 * t];
    twA[16 + t] = tw[512 - 32 * t];
    twB[t] = tw[(2048 - 32 * t) & (N - 1)];
    twB[16 + t] = tw[(32 * t + 1536) & (N - 1)];
  }
  const __nv_bfloat16* base = (tensor ? values : keys) + (int64_t)c * ld_chunk +
                              (int64_t)l * ld_layer + (int64_t)group * SIG_PER_CTA * 2;
  constexpr int NACC = 32 / SIG;
  float acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = 0.f;
  // batch b's 2 SIG lanes of every token (SIG * 4 bytes): SIG / 4 threads
  // per token row, 16 bytes each, 256 rows per pass
  constexpr int PIECES = SIG / 4;
  auto prefetch = [&](int b) {
    const int piece = t % PIECES, row = t / PIECES;
    const __nv_bfloat16* src = base + b * SIG * 2 + piece * 8 + (int64_t)row * ld_token;
    uint32_t* dst = stg + row * SIG + piece * 4;
    const int64_t step = (int64_t)(TH / PIECES) * ld_token;
#pragma unroll 1
    for (int i = 0; i < N / (TH / PIECES); ++i) {
      cp_async16(dst, src);
      src += step;
      dst += (TH / PIECES) * SIG;
    }
    cp_async_commit();
  };
  prefetch(0);
  // step-2 role: row k1 = q >> 1, half h = q & 1 (partner lane t ^ SIG)
  const int h = q & 1, k1r = q >> 1;
  const float sg = h ? -1.f : 1.f;
  const bool cut0 = h && k1r == 0;  // k = 3N/4 (k1 = 0, k2 = 48) is cut
  __syncthreads();

#pragma unroll 1
  for (int b = 0; b < S::BATCHES; ++b) {
    cp_async_wait_all();
    __syncthreads();
    // ---- step 1: 32-point DFT over n1 of tokens q + 64 n1, twiddle, exchange
    {
      const int n2 = q;
      cf v[32];
#pragma unroll
      for (int n1 = 0; n1 < 32; ++n1) v[n1] = unpack_bf16x2(stg[(n2 + 64 * n1) * SIG + s]);
      fwd<32>(v);
#pragma unroll
      for (int p = 0; p < 32; ++p) {
        const int k1 = digrev<32>(p);
        xb[S::xi(s, k1, n2)] = cmul(v[p], T[(n2 * k1) & (N - 1)]);
      }
    }
    __syncthreads();
    if (b + 1 < S::BATCHES) prefetch(b + 1);
    // ---- step 2: half of row k1r per lane: 32-point DFT of u[2m + h], band
    // combine over the lane pair, inverse split, 32-point inverse, twiddle
    {
      cf v[32];
#pragma unroll
      for (int m = 0; m < 32; ++m) {
        v[m] = xb[S::xi(s, k1r, 2 * m + h)];
        if (m & 1) v[m] = __fmul2_rn(v[m], make_float2(sg, sg));
      }
      fwd<32>(v);
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        const cf r = shfl_xor_cf(v[posof32(16 + kk)], SIG);
        v[posof32(kk)] = v[posof32(kk)] + cmul(r, twA[16 * h + kk]);
      }
      if (cut0) v[posof32(0)] = make_float2(0.f, 0.f);
#pragma unroll
      for (int kk = 0; kk < 16; ++kk)
        v[posof32(16 + kk)] = shfl_xor_cf(cmul(v[posof32(kk)], twB[16 * h + kk]), SIG);
      inv<32>(v);
#pragma unroll
      for (int m = 0; m < 32; ++m) {
        const int n2 = 2 * m + h;
        xb[S::xi(s, k1r, n2)] = cmulc(v[m], T[(n2 * k1r) & (N - 1)]);
      }
    }
    __syncthreads();
    // ---- step 3: 32-point inverse over k1 -> tokens q + 64 n1', energies
    float e[32];
    {
      const int n2 = q;
      cf w[32];
#pragma unroll
      for (int p = 0; p < 32; ++p) w[p] = xb[S::xi(s, digrev<32>(p), n2)];
      inv<32>(w);
#pragma unroll
      for (int n1 = 0; n1 < 32; ++n1) e[n1] = fmaf(w[n1].x, w[n1].x, w[n1].y * w[n1].y);
    }
    // reduce-scatter over the SIG slots (xor SIG/2 ... 1): lane s ends with
    // n1 in [NACC s, NACC s + NACC)
#pragma unroll
    for (int lv = SIG / 2, len = 16; lv >= 1; lv >>= 1, len >>= 1) {
      const bool up = s & lv;
#pragma unroll
      for (int i = 0; i < len; ++i) {
        const float send = up ? e[i] : e[len + i];
        e[i] = (up ? e[len + i] : e[i]) + __shfl_xor_sync(0xffffffffu, send, lv);
      }
    }
#pragma unroll
    for (int i = 0; i < NACC; ++i) acc[i] += e[i];
  }
  float* out = partial + ((((int64_t)c * L + l) * 2 + tensor) * groups + group) * N;
#pragma unroll
  for (int i = 0; i < NACC; ++i) out[q + 64 * (NACC * s + i)] = acc[i];
}

__global__ void fs_twiddle(float2* tw) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= N) return;
  double sn, cs;
  sincospi(2.0 * (double)m / (double)N, &sn, &cs);
  tw[m] = make_float2((float)cs, (float)-sn);  // W_N^m = exp(-2 pi i m / N)
}

// layer score = 0.5 sqrt(EK) / N + 0.5 sqrt(EV) / N (f64, groups summed in
// order), aggregate = sequential layer sum / L (ct/spectral.py:74-78,156)
__global__ void fs_combine(const float* __restrict__ partial, int C, int L, int groups,
                           double* __restrict__ layer_scores, double* __restrict__ agg) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)C * N) return;
  const int c = (int)(i / N), n = (int)(i % N);
  double acc = 0.0;
  for (int l = 0; l < L; ++l) {
    double e[2];
    for (int t = 0; t < 2; ++t) {
      const float* p = partial + (((int64_t)c * L + l) * 2 + t) * groups * N + n;
      double s = 0.0;
      for (int g = 0; g < groups; ++g) s += (double)p[(int64_t)g * N];
      e[t] = s;
    }
    const double sc = 0.5 * (sqrt(e[0]) / (double)N) + 0.5 * (sqrt(e[1]) / (double)N);
    if (layer_scores) layer_scores[((int64_t)c * L + l) * N + n] = sc;
    acc += sc;
  }
  agg[i] = acc / (double)L;
}

// Per chunk: certify the boundary between order positions k-1 and k, or mark
// the window of positions whose scores could cross it.  win[c] = {p0, p1}
// (p1 < p0: certified / no boundary); wcount[c] = window size (0 certified,
// > WMAX: too wide, the host re-scores the chunk exactly).
__global__ void fs_window(const double* __restrict__ agg, const int32_t* __restrict__ order,
                          int C, int k, double g, int2* __restrict__ win,
                          int32_t* __restrict__ wcount) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const double* a = agg + (int64_t)c * N;
  const int32_t* o = order + (int64_t)c * N;
  int2 w = make_int2(1, 0);
  int cnt = 0;
  if (k > 0 && k < N) {
    const double ak = a[o[k - 1]], ak1 = a[o[k]];
    if (!(ak * (1.0 - g) > ak1 * (1.0 + g))) {
      const double vhi = ak * (1.0 + g) / (1.0 - g), vlo = ak1 * (1.0 - g) / (1.0 + g);
      int p0 = k - 1, p1 = k;
      while (p0 > 0 && a[o[p0 - 1]] <= vhi) --p0;
      while (p1 < N - 1 && a[o[p1 + 1]] >= vlo) ++p1;
      w = make_int2(p0, p1);
      cnt = p1 - p0 + 1;
    }
  }
  win[c] = w;
  wcount[c] = cnt;
}

// p[m] = (1/N) sum_{k in band} w_k cos(2 pi k m / N): row of P = F^-1 M F
__global__ void fs_kernel_row(int cutoff, int high, double* p) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= N) return;
  const int klo = high ? cutoff : 0, khi = high ? N / 2 : min(cutoff - 1, N / 2);
  double s = 0.0;
  for (int k = klo; k <= khi; ++k) {
    const int km = (int)(((long long)k * m) % N);
    s += ((k == 0 || 2 * k == N) ? 1.0 : 2.0) * cospi(2.0 * (double)km / (double)N);
  }
  p[m] = s / (double)N;
}

// Exact (float64) energy of the window tokens of one (chunk, layer, tensor):
// y_w[lane] = sum_n p[(i_w - n) mod N] x[n][lane], E_w = sum_lanes y_w^2.
// grid: x = chunk (chunks without a re-score window exit), y = 2 layer +
// tensor, z = group of RS_LANES lanes (so a windowed chunk spreads over
// 2 L (lanes / RS_LANES) small CTAs); R in {2, 4, 6, 8} window tokens per pass
// (one pass over the rows serves R tokens); the warp-uniform p values are
// shared-memory broadcasts.  Each CTA writes its partial energies to its own
// slot; fs_fixup sums the groups in a fixed order (deterministic).
constexpr int RS_THREADS = 64, RS_LPT = 4, RS_UNROLL = 8;
constexpr int RS_LANES = RS_THREADS * RS_LPT;
template <typename IN>
__device__ __forceinline__ float4 load4(const IN* p);
template <>
__device__ __forceinline__ float4 load4<__nv_bfloat16>(const __nv_bfloat16* p) {
  const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
  return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u),
                     __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xffff0000u));
}
template <>
__device__ __forceinline__ float4 load4<float>(const float* p) {
  return __ldg(reinterpret_cast<const float4*>(p));
}
template <int R, typename IN>
__device__ __forceinline__ void rescore_pass(const IN* __restrict__ x, int lanes, int64_t ld_token,
                                             const double* ps, const int* tok, int nr,
                                             double (*red)[8], double* out) {
  double part[R];
#pragma unroll
  for (int r = 0; r < R; ++r) part[r] = 0.0;
  for (int lane0 = threadIdx.x * RS_LPT; lane0 < lanes; lane0 += RS_LANES) {
    double y[R][RS_LPT];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int i = 0; i < RS_LPT; ++i) y[r][i] = 0.0;
    for (int n0 = 0; n0 < N; n0 += RS_UNROLL) {
      float4 xv[RS_UNROLL];  // RS_UNROLL rows in flight
#pragma unroll
      for (int u = 0; u < RS_UNROLL; ++u) xv[u] = load4<IN>(x + (int64_t)(n0 + u) * ld_token + lane0);
#pragma unroll
      for (int u = 0; u < RS_UNROLL; ++u) {
        const double x4[RS_LPT] = {(double)xv[u].x, (double)xv[u].y, (double)xv[u].z,
                                   (double)xv[u].w};
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double pv = ps[(tok[r] - n0 - u) & (N - 1)];
#pragma unroll
          for (int i = 0; i < RS_LPT; ++i) y[r][i] = fma(pv, x4[i], y[r][i]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int i = 0; i < RS_LPT; ++i) part[r] = fma(y[r][i], y[r][i], part[r]);
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    double v = part[r];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][r] = v;
  }
  __syncthreads();
  if ((int)threadIdx.x < nr) {
    double v = 0.0;
    for (int wi = 0; wi < RS_THREADS / 32; ++wi) v += red[wi][threadIdx.x];
    out[threadIdx.x] = v;
  }
  __syncthreads();
}
template <typename IN>
__global__ void __launch_bounds__(RS_THREADS)
fs_rescore(const IN* __restrict__ keys, const IN* __restrict__ values, int L, int lanes,
           int64_t ld_token, int64_t ld_layer, int64_t ld_chunk, const double* __restrict__ p,
           const int2* __restrict__ win, const int32_t* __restrict__ wcount,
           const int32_t* __restrict__ order, double* __restrict__ wpart) {
  const int c = blockIdx.x;
  const int W = wcount[c];
  if (W <= 0 || W > WMAX) return;
  __shared__ double ps[N];
  __shared__ double red[RS_THREADS / 32][8];  // [warp][token]
  __shared__ double res[8];
  const int l = blockIdx.y >> 1, tensor = blockIdx.y & 1, g = blockIdx.z, groups = gridDim.z;
  const int2 w = win[c];
  for (int i = threadIdx.x; i < N; i += RS_THREADS) ps[i] = p[i];
  __syncthreads();
  const int lane_lo = g * RS_LANES, n_lanes = min(RS_LANES, lanes - lane_lo);
  const IN* x = (tensor ? values : keys) + (int64_t)c * ld_chunk + (int64_t)l * ld_layer + lane_lo;
  for (int r0 = 0; r0 < W; r0 += 8) {
    const int nr = min(8, W - r0);
    int tok[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) tok[r] = r < nr ? order[(int64_t)c * N + w.x + r0 + r] : 0;
    if (nr <= 2)
      rescore_pass<2, IN>(x, n_lanes, ld_token, ps, tok, nr, red, res);
    else if (nr <= 4)
      rescore_pass<4, IN>(x, n_lanes, ld_token, ps, tok, nr, red, res);
    else if (nr <= 6)
      rescore_pass<6, IN>(x, n_lanes, ld_token, ps, tok, nr, red, res);
    else
      rescore_pass<8, IN>(x, n_lanes, ld_token, ps, tok, nr, red, res);
    if ((int)threadIdx.x < nr)
      wpart[((((int64_t)c * WMAX + r0 + threadIdx.x) * L + l) * 2 + tensor) * groups + g] =
          res[threadIdx.x];
  }
}

// Exact window scores -> window re-ordered by (score desc, index asc).
__global__ void fs_fixup(int C, const int2* __restrict__ win, const int32_t* __restrict__ wcount,
                         const double* __restrict__ wpart, int groups, int L,
                         int32_t* __restrict__ order, double* __restrict__ agg) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C || wcount[c] <= 0 || wcount[c] > WMAX) return;
  const int slot = c;
  const int2 w = win[c];
  const int W = w.y - w.x + 1;
  int32_t* o = order + (int64_t)c * N + w.x;
  double sc[WMAX];
  int id[WMAX];
  for (int r = 0; r < W; ++r) {
    double acc = 0.0;
    for (int l = 0; l < L; ++l) {
      double e[2];
      for (int t = 0; t < 2; ++t) {  // lane groups summed in order
        const double* q = wpart + ((((int64_t)slot * WMAX + r) * L + l) * 2 + t) * groups;
        double v = 0.0;
        for (int g = 0; g < groups; ++g) v += q[g];
        e[t] = v;
      }
      acc += 0.5 * sqrt(e[0]) + 0.5 * sqrt(e[1]);
    }
    sc[r] = acc / (double)L;
    id[r] = o[r];
  }
  for (int i = 1; i < W; ++i) {  // insertion sort: desc score, asc index
    const double s = sc[i];
    const int t = id[i];
    int j = i - 1;
    while (j >= 0 && (sc[j] < s || (sc[j] == s && id[j] > t))) {
      sc[j + 1] = sc[j];
      id[j + 1] = id[j];
      --j;
    }
    sc[j + 1] = s;
    id[j + 1] = t;
  }
  for (int r = 0; r < W; ++r) {
    o[r] = id[r];
    agg[(int64_t)c * N + id[r]] = sc[r];
  }
}

}  // namespace fs
}  // namespace ct

using namespace ct;

extern "C" int ct_desc_order(const double* scores, int64_t rows, int64_t n, int32_t* order,
                             void* stream);

static size_t fs_groups(int64_t lanes) { return (size_t)(lanes / (2 * fs::SIG_PER_CTA)); }
static size_t fs_rs_groups(int64_t lanes) { return (size_t)((lanes + fs::RS_LANES - 1) / fs::RS_LANES); }

extern "C" size_t ct_score_fast_workspace_bytes(int64_t C, int64_t L, int64_t N, int64_t lanes) {
  if (N != fs::N || lanes % (2 * fs::SIG_PER_CTA)) return 0;
  size_t b = align_up((size_t)C * L * 2 * fs_groups(lanes) * N * sizeof(float), 256);
  b += align_up((size_t)N * sizeof(float2), 256);                 // twiddles
  b += align_up((size_t)N * sizeof(double), 256);                 // projection row
  b += align_up((size_t)C * sizeof(int2), 256);                   // windows
  b += align_up((size_t)C * fs::WMAX * L * 2 * fs_rs_groups(lanes) * sizeof(double), 256);  // window energies
  return b;
}

extern "C" int ct_score_select_fast(const void* keys, const void* values, int dtype, int64_t C,
                                    int64_t L, int64_t N, int64_t lanes, int64_t ld_token,
                                    int64_t ld_layer, int64_t ld_chunk, int64_t cutoff, int band,
                                    int64_t k, double guard, double* layer_scores,
                                    double* agg_scores, int32_t* agg_order, int32_t* wcount,
                                    void* workspace, size_t workspace_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (C < 1 || L < 1 || lanes < 1)
    return fail(CT_ERR_SHAPE, "score geometry C=%lld L=%lld lanes=%lld", (long long)C,
                (long long)L, (long long)lanes);
  if (N != fs::N || lanes % (2 * fs::SIG_PER_CTA))
    return fail(CT_ERR_UNSUPPORTED, "fast scorer needs N = %d and lanes %% %d == 0 (N=%lld)",
                fs::N, 2 * fs::SIG_PER_CTA, (long long)N);
  if (!valid_dtype(dtype)) return fail(CT_ERR_PARAM, "dtype %d", dtype);
  {
    // the window re-score reads 4 lanes per load: 8-byte (bf16) / 16-byte
    // (f32) aligned rows
    const int64_t vec = 4;  // elements per load
    const uintptr_t abytes = dtype == CT_BF16 ? 8 : 16;
    if ((((uintptr_t)keys | (uintptr_t)values) & (abytes - 1)) || ld_token % vec ||
        ld_layer % vec || ld_chunk % vec)
      return fail(CT_ERR_UNSUPPORTED, "fast scorer needs %d-byte aligned rows",
                  (int)abytes);
  }
  if (band != 0 && band != 1) return fail(CT_ERR_PARAM, "band %d", band);
  if (cutoff < 0 || cutoff > N / 2 + 1) return fail(CT_ERR_PARAM, "cutoff %lld", (long long)cutoff);
  if (k < 0 || k > N) return fail(CT_ERR_PARAM, "k %lld", (long long)k);
  if (!(guard >= 0.0 && guard < 0.5)) return fail(CT_ERR_PARAM, "guard %g", guard);
  if (!keys || !values || !agg_scores || !agg_order || !wcount)
    return fail(CT_ERR_PARAM, "null tensor");
  if (C * L > 65535) return fail(CT_ERR_UNSUPPORTED, "C*L too large");
  if (workspace_bytes < ct_score_fast_workspace_bytes(C, L, N, lanes))
    return fail(CT_ERR_PARAM, "workspace too small");
  const int groups = (int)fs_groups(lanes);
  char* ws = (char*)workspace;
  float* partial = (float*)ws;
  ws += align_up((size_t)C * L * 2 * groups * N * sizeof(float), 256);
  float2* tw = (float2*)ws;
  ws += align_up((size_t)N * sizeof(float2), 256);
  double* prow = (double*)ws;
  ws += align_up((size_t)N * sizeof(double), 256);
  int2* win = (int2*)ws;
  ws += align_up((size_t)C * sizeof(int2), 256);
  double* wenergy = (double*)ws;
  int rc;
  fs::fs_twiddle<<<(fs::N + 255) / 256, 256, 0, st>>>(tw);
  if ((rc = check_launch("fs_twiddle"))) return rc;
  const size_t smem = (size_t)fs::SIG_PER_BATCH * 32 * 64 * sizeof(fs::cf) + fs::N * sizeof(fs::cf);
  dim3 grid((unsigned)groups, 2, (unsigned)(C * L));
  const bool aligned16 = !(((uintptr_t)keys | (uintptr_t)values) & 15) && ld_token % 8 == 0 &&
                         ld_layer % 8 == 0 && ld_chunk % 8 == 0;
  const bool lb = band == 0 && cutoff == fs::N / 4;
  if (dtype == CT_BF16 && aligned16 && lb) {
    // one 512-thread CTA per SM (SIG = 8); two 256-thread CTAs per SM
    // (SIG = 4) measured 3 % slower (profiles/round2_scorer_split_ncu.md)
    auto kern = fs::fs_energy_split_kernel<8>;
    CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)fs::Split<8>::SMEM));
    kern<<<grid, fs::Split<8>::THREADS, fs::Split<8>::SMEM, st>>>(
        (const __nv_bfloat16*)keys, (const __nv_bfloat16*)values, (int)L, ld_token, ld_layer,
        ld_chunk, tw, groups, partial);
  } else if (dtype == CT_BF16 && aligned16) {
    auto kern = lb ? fs::fs_energy_kernel<__nv_bfloat16, true, true>
                   : fs::fs_energy_kernel<__nv_bfloat16, true, false>;
    const size_t smem_st = smem + fs::STAGE_BYTES;
    CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_st));
    kern<<<grid, fs::THREADS, smem_st, st>>>((const __nv_bfloat16*)keys,
                                             (const __nv_bfloat16*)values, (int)L, ld_token,
                                             ld_layer, ld_chunk, (int)cutoff, band, tw, groups,
                                             partial);
  } else if (dtype == CT_BF16) {
    auto kern = fs::fs_energy_kernel<__nv_bfloat16, false, false>;
    CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, fs::THREADS, smem, st>>>((const __nv_bfloat16*)keys, (const __nv_bfloat16*)values,
                                          (int)L, ld_token, ld_layer, ld_chunk, (int)cutoff, band,
                                          tw, groups, partial);
  } else {
    auto kern = fs::fs_energy_kernel<float, false, false>;
    CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, fs::THREADS, smem, st>>>((const float*)keys, (const float*)values, (int)L,
                                          ld_token, ld_layer, ld_chunk, (int)cutoff, band, tw,
                                          groups, partial);
  }
  if ((rc = check_launch("fs_energy_kernel"))) return rc;
  fs::fs_combine<<<(unsigned)((C * fs::N + 255) / 256), 256, 0, st>>>(partial, (int)C, (int)L,
                                                                      groups, layer_scores,
                                                                      agg_scores);
  if ((rc = check_launch("fs_combine"))) return rc;
  if ((rc = ct_desc_order(agg_scores, C, N, agg_order, stream))) return rc;
  fs::fs_window<<<(unsigned)((C + 127) / 128), 128, 0, st>>>(agg_scores, agg_order, (int)C,
                                                             (int)k, guard, win, wcount);
  if ((rc = check_launch("fs_window"))) return rc;
  // every chunk gets re-score CTAs; the ones without a window (or with one
  // wider than FS_WMAX, which the caller re-scores exactly) exit at once, so
  // the call never waits for the window counts on the host
  fs::fs_kernel_row<<<(fs::N + 255) / 256, 256, 0, st>>>((int)cutoff, band, prow);
  if ((rc = check_launch("fs_kernel_row"))) return rc;
  const int rs_groups = (int)fs_rs_groups(lanes);
  if (2 * L > 65535) return fail(CT_ERR_UNSUPPORTED, "2 L too large for the re-score grid");
  dim3 rgrid((unsigned)C, (unsigned)(2 * L), (unsigned)rs_groups);
  if (dtype == CT_BF16)
    fs::fs_rescore<__nv_bfloat16><<<rgrid, fs::RS_THREADS, 0, st>>>(
        (const __nv_bfloat16*)keys, (const __nv_bfloat16*)values, (int)L, (int)lanes, ld_token,
        ld_layer, ld_chunk, prow, win, wcount, agg_order, wenergy);
  else
    fs::fs_rescore<float><<<rgrid, fs::RS_THREADS, 0, st>>>((const float*)keys, (const float*)values, (int)L,
                                                 (int)lanes, ld_token, ld_layer, ld_chunk, prow,
                                                 win, wcount, agg_order, wenergy);
  if ((rc = check_launch("fs_rescore"))) return rc;
  fs::fs_fixup<<<(unsigned)((C + 63) / 64), 64, 0, st>>>((int)C, win, wcount, wenergy, rs_groups, (int)L,
                                                         agg_order, agg_scores);
  return check_launch("fs_fixup");
}
