// (1) Frequency-domain critical-token scorer + deterministic ordering +
// selection plan.  Replaces ct/spectral.py:69-90 (_band_scores /
// low_freq_scores), :149-159 (rank_chunk), :99-101 (_descending_order),
// :162-184 (selection) and the global assembly of ct/toymodel.py:246-267.
//
// Design (B200): the token axis of every (head, dim) lane is a real signal.
// Two lanes are packed into one complex signal z = x_a + i x_b; because the
// low-pass keeps a Hermitian-symmetric bin set, lowpass(z) = lowpass(x_a) +
// i lowpass(x_b), so one complex FFT pair scores two lanes.  A CTA owns one
// (chunk, layer, tensor, 128-lane block); it streams lane groups through a
// shared-memory Stockham FFT (radix 8/4/2 passes, natural order, twiddles
// from a float64 table), masks bins with min(k, N-k) >= c on the first
// inverse pass, and accumulates |recon|^2 per token in registers across lane
// groups.  Partial per-token energies of the lane blocks are combined in a
// fixed order (deterministic), square-rooted, averaged over K/V and summed
// sequentially over layers exactly as ct/spectral.py:74-78,156 do.  Orders
// are a block bitonic sort on (score desc, index asc) == numpy's stable
// argsort of -scores.  Non power-of-two N uses a direct circulant projection
// (same math, O(N^2) per lane).
#include "common.cuh"

namespace ct {

template <typename T> struct cpx { T x, y; };

template <typename T>
__device__ __forceinline__ cpx<T> cmul(cpx<T> a, cpx<T> b) {
  return {a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x};
}
template <typename T>
__device__ __forceinline__ cpx<T> cadd(cpx<T> a, cpx<T> b) { return {a.x + b.x, a.y + b.y}; }
template <typename T>
__device__ __forceinline__ cpx<T> csub(cpx<T> a, cpx<T> b) { return {a.x - b.x, a.y - b.y}; }
// multiply by -i (forward) or +i (inverse)
template <bool INV, typename T>
__device__ __forceinline__ cpx<T> mul_mi(cpx<T> a) {
  return INV ? cpx<T>{-a.y, a.x} : cpx<T>{a.y, -a.x};
}

template <int R, bool INV, typename T>
__device__ __forceinline__ void dft_small(cpx<T>* v) {
  if constexpr (R == 2) {
    cpx<T> a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  } else if constexpr (R == 4) {
    cpx<T> t0 = cadd(v[0], v[2]), t1 = csub(v[0], v[2]);
    cpx<T> t2 = cadd(v[1], v[3]), t3 = mul_mi<INV>(csub(v[1], v[3]));
    v[0] = cadd(t0, t2);
    v[2] = csub(t0, t2);
    v[1] = cadd(t1, t3);
    v[3] = csub(t1, t3);
  } else {  // R == 8: radix-2 split into two radix-4 DFTs
    cpx<T> e[4] = {v[0], v[2], v[4], v[6]};
    cpx<T> o[4] = {v[1], v[3], v[5], v[7]};
    dft_small<4, INV>(e);
    dft_small<4, INV>(o);
    const T h = (T)0.70710678118654752440;
    // W8^k = exp(-/+ i pi k / 4)
    cpx<T> w1 = INV ? cpx<T>{h, h} : cpx<T>{h, -h};
    cpx<T> w3 = INV ? cpx<T>{-h, h} : cpx<T>{-h, -h};
    cpx<T> o1 = cmul(o[1], w1);
    cpx<T> o2 = mul_mi<INV>(o[2]);
    cpx<T> o3 = cmul(o[3], w3);
    v[0] = cadd(e[0], o[0]);
    v[4] = csub(e[0], o[0]);
    v[1] = cadd(e[1], o1);
    v[5] = csub(e[1], o1);
    v[2] = cadd(e[2], o2);
    v[6] = csub(e[2], o2);
    v[3] = cadd(e[3], o3);
    v[7] = csub(e[3], o3);
  }
}

template <typename T> struct ScoreCfg;
// S complex signals (2S lanes) in flight per CTA; S*N*sizeof(cpx<T>) = 128 KiB.
template <> struct ScoreCfg<double> { static constexpr int POINTS = 8192; };
template <> struct ScoreCfg<float> { static constexpr int POINTS = 8192; };

constexpr int SCORE_THREADS = 1024;
constexpr int LANE_BLOCK = 128;

__host__ __device__ constexpr int pass_radix(int logn, int p) {
  // radix-8 passes first, then one radix-4 or radix-2 pass for the rest
  return (p < logn / 3) ? 8 : (1 << (logn % 3));
}
__host__ __device__ constexpr int num_passes(int logn) { return logn / 3 + (logn % 3 ? 1 : 0); }

// Shared-memory signal index with one pad element per 8: keeps the stride-R
// stores of the first Stockham pass off a single bank.
__device__ __forceinline__ int spad(int i) { return i + (i >> 3); }

template <typename IN>
__device__ __forceinline__ double load_as_double(const IN* p) { return (double)to_f32(*p); }
__device__ __forceinline__ double load_as_double(const float* p) { return (double)*p; }

// One Stockham pass over all S signals in shared memory (in place: every
// thread loads all its butterflies, barrier, then stores).  MASK applies the
// low-pass on the loaded (natural-order) bins; ENERGY stores |z|^2 into .x
// instead of z (the last inverse pass feeds the per-token accumulation).
template <typename T, int LOGN, int R, bool INV, bool MASK, bool ENERGY>
__device__ __forceinline__ void stockham_pass(cpx<T>* sig, int S, int Ns,
                                              const cpx<T>* __restrict__ tw,
                                              int cutoff) {
  constexpr int N = 1 << LOGN;
  constexpr int NB = N / R;  // butterflies per signal
  constexpr int PTS = ScoreCfg<T>::POINTS;
  constexpr int BPT = (PTS / R + SCORE_THREADS - 1) / SCORE_THREADS;
  cpx<T> v[BPT][R];
  const int total = S * NB;
  const int step = N / (Ns * R);
#pragma unroll
  for (int k = 0; k < BPT; ++k) {
    const int b = threadIdx.x + k * SCORE_THREADS;
    if (b < total) {
      const int sg = b / NB, j = b % NB;
      const int jm = j % Ns;
      // twiddles w^r by recurrence from one table load (fewer LSU ops; the
      // extra complex multiplies run on the otherwise idle FP pipes)
      cpx<T> w1 = {(T)1, (T)0};
      if (jm > 0) {
        w1 = tw[jm * step];
        if (INV) w1.y = -w1.y;
      }
      cpx<T> wr = w1;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int idx = j + r * NB;
        cpx<T> val = sig[spad(sg * N + idx)];
        if (MASK) {
          const int kk = idx < N - idx ? idx : N - idx;
          // cutoff >= 0: low band keeps min(k,N-k) < c; cutoff = -(c+1): high band
          if (cutoff >= 0 ? kk >= cutoff : kk < -cutoff - 1) val = {(T)0, (T)0};
        }
        if (r > 0) {
          val = cmul(val, wr);
          wr = cmul(wr, w1);
        }
        v[k][r] = val;
      }
      dft_small<R, INV>(v[k]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < BPT; ++k) {
    const int b = threadIdx.x + k * SCORE_THREADS;
    if (b < total) {
      const int sg = b / NB, j = b % NB;
      const int idxD = (j / Ns) * Ns * R + (j % Ns);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (ENERGY)
          sig[spad(sg * N + idxD + r * Ns)].x = v[k][r].x * v[k][r].x + v[k][r].y * v[k][r].y;
        else
          sig[spad(sg * N + idxD + r * Ns)] = v[k][r];
      }
    }
  }
  __syncthreads();
}

template <int LOGN, int P>
__host__ __device__ constexpr int ns_before() {
  if constexpr (P == 0) return 1;
  else return ns_before<LOGN, P - 1>() * pass_radix(LOGN, P - 1);
}

template <typename T, int LOGN, int P, bool INV>
__device__ __forceinline__ void run_passes(cpx<T>* sig, int S, const cpx<T>* tw, int cutoff) {
  if constexpr (P < num_passes(LOGN)) {
    constexpr int R = pass_radix(LOGN, P);
    constexpr bool LAST = P == num_passes(LOGN) - 1;
    stockham_pass<T, LOGN, R, INV, INV && P == 0, INV && LAST>(sig, S, ns_before<LOGN, P>(), tw,
                                                               cutoff);
    run_passes<T, LOGN, P + 1, INV>(sig, S, tw, cutoff);
  }
}

// grid: x = lane block, y = tensor (0 K, 1 V), z = c*L + l.  Per lane group
// (2S lanes): load -> forward FFT -> masked inverse FFT -> |recon|^2 in place
// -> per-token sums over the S signals in fixed order into registers.
template <typename T, typename IN, int LOGN>
__global__ void __launch_bounds__(SCORE_THREADS, 1)
fft_energy_kernel(const IN* __restrict__ keys, const IN* __restrict__ values,
                  int L, int lanes, int64_t ld_token, int64_t ld_layer,
                  int64_t ld_chunk, int cutoff, const cpx<T>* __restrict__ tw,
                  double* __restrict__ partial) {
  constexpr int N = 1 << LOGN;
  constexpr int PTS = ScoreCfg<T>::POINTS;
  constexpr int S = PTS / N < 1 ? 1 : (PTS / N > 64 ? 64 : PTS / N);
  constexpr int TPT = (N + SCORE_THREADS - 1) / SCORE_THREADS;  // tokens per thread
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cpx<T>* sig = reinterpret_cast<cpx<T>*>(smem_raw);

  const int lb = blockIdx.x, tensor = blockIdx.y;
  const int c = blockIdx.z / L, l = blockIdx.z % L;
  const IN* base = (tensor == 0 ? keys : values) + (int64_t)c * ld_chunk + (int64_t)l * ld_layer;
  const int lane0 = lb * LANE_BLOCK;
  const int lane_end = min(lanes, lane0 + LANE_BLOCK);

  double acc[TPT];
#pragma unroll
  for (int i = 0; i < TPT; ++i) acc[i] = 0.0;

  for (int g0 = lane0; g0 < lane_end; g0 += 2 * S) {
    // load 2S lanes of every token: one thread per (token, 8-lane slice) with
    // a 16-B (bf16) / 2x16-B (f32) vector load when the slice is in range;
    // smem writes are then contiguous per signal (conflict-free).
    constexpr int SL = 4;  // signals per slice (8 lanes)
    const bool vec_ok = ((ld_token * (int64_t)sizeof(IN)) % 16 == 0) &&
                        (((uintptr_t)base) % 16 == 0) && (g0 % 8 == 0);
    for (int q = threadIdx.x; q < (S / SL > 0 ? S / SL : 1) * N; q += SCORE_THREADS) {
      const int n = q % N, sl = q / N;
      const IN* row = base + (int64_t)n * ld_token;
      const int lbase = g0 + 8 * sl;
      if (S >= SL && vec_ok && lbase + 8 <= lane_end) {
        float f[8];
        if constexpr (sizeof(IN) == 2) {
          const uint4 u = __ldg(reinterpret_cast<const uint4*>(row + lbase));
          const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float2 ff = __bfloat1622float2(h2[t]);
            f[2 * t] = ff.x;
            f[2 * t + 1] = ff.y;
          }
        } else {
          const float4 a = __ldg(reinterpret_cast<const float4*>(row + lbase));
          const float4 b = __ldg(reinterpret_cast<const float4*>(row + lbase) + 1);
          f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
          f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
        }
#pragma unroll
        for (int t = 0; t < SL; ++t)
          sig[spad((sl * SL + t) * N + n)] = {(T)f[2 * t], (T)f[2 * t + 1]};
      } else {
        const int smax = S >= SL ? SL : S;
        for (int t = 0; t < smax; ++t) {
          const int la = lbase + 2 * t, lbn = la + 1;
          T re = la < lane_end ? (T)load_as_double(row + la) : (T)0;
          T im = lbn < lane_end ? (T)load_as_double(row + lbn) : (T)0;
          sig[spad((sl * SL + t) * N + n)] = {re, im};
        }
      }
    }
    __syncthreads();
    run_passes<T, LOGN, 0, false>(sig, S, tw, cutoff);
    run_passes<T, LOGN, 0, true>(sig, S, tw, cutoff);
    // energies now in sig[s][n].x: fixed-order sum over the group's signals
#pragma unroll
    for (int i = 0; i < TPT; ++i) {
      const int n = threadIdx.x + i * SCORE_THREADS;
      if (n < N) {
        double e = 0.0;
        for (int sg = 0; sg < S; ++sg) e += (double)sig[spad(sg * N + n)].x;
        acc[i] += e;
      }
    }
    __syncthreads();
  }
  const double inv_n2 = 1.0 / ((double)N * (double)N);
  const int nlb = gridDim.x;
  double* out = partial + ((((int64_t)blockIdx.z * 2 + tensor) * nlb) + lb) * N;
#pragma unroll
  for (int i = 0; i < TPT; ++i) {
    const int n = threadIdx.x + i * SCORE_THREADS;
    if (n < N) out[n] = acc[i] * inv_n2;
  }
}

// ---------------------------------------------------------------------------
// v2 energy kernel for N = 256*R3 (512..4096): register-resident Stockham FFT.
//
// A group of GT = N/16 threads owns one packed signal (2 lanes); every thread
// holds 16 complex points in registers.  Forward radices (16, 16, R3), inverse
// (R3, 16, 16): the forward's last pass leaves thread t holding exactly the
// bins j + (N/R3) r its inverse first pass needs, so the low-pass mask and the
// spectrum never touch shared memory.  Four exchanges per signal (f1->f2,
// f2->f3, i1->i2, i2->i3) go through a padded per-group buffer; the inverse's
// last pass leaves token t + GT r in register r, so |recon|^2 accumulates in
// registers over all of the CTA's signals.  Input lanes arrive as a [N][2*NG]
// tile staged with cp.async one tile ahead.  Twiddles: W^a, W^2a, W^4a, W^8a
// from the table, the other powers as products (depth <= 3).
// ---------------------------------------------------------------------------
constexpr int FFT2_THREADS = 512;

template <typename T> struct tconst;
template <> struct tconst<double> {
  static constexpr double h = 0.70710678118654752440, c1 = 0.92387953251128675613,
                          s1 = 0.38268343236508977173;
};
template <> struct tconst<float> {
  static constexpr float h = 0.70710678118654752440f, c1 = 0.92387953251128675613f,
                         s1 = 0.38268343236508977173f;
};

// 16-point DFT in place, natural order in and out (4 x 4 with W16 twiddles).
template <bool INV, typename T>
__device__ __forceinline__ void dft16(cpx<T>* v) {
  cpx<T> a[4][4];
#pragma unroll
  for (int n1 = 0; n1 < 4; ++n1) {
    cpx<T> t[4] = {v[n1], v[n1 + 4], v[n1 + 8], v[n1 + 12]};
    dft_small<4, INV>(t);
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) a[n1][k2] = t[k2];
  }
  const T h = tconst<T>::h, c1 = tconst<T>::c1, s1 = tconst<T>::s1;
  const T sg = INV ? (T)1 : (T)-1;  // sign of the imaginary part of W16^1
  // W16^e for e = n1*k2
  a[1][1] = cmul(a[1][1], cpx<T>{c1, sg * s1});
  a[1][2] = cmul(a[1][2], cpx<T>{h, sg * h});
  a[1][3] = cmul(a[1][3], cpx<T>{s1, sg * c1});
  a[2][1] = cmul(a[2][1], cpx<T>{h, sg * h});
  a[2][2] = mul_mi<INV>(a[2][2]);
  a[2][3] = cmul(a[2][3], cpx<T>{-h, sg * h});
  a[3][1] = cmul(a[3][1], cpx<T>{s1, sg * c1});
  a[3][2] = cmul(a[3][2], cpx<T>{-h, sg * h});
  a[3][3] = cmul(a[3][3], cpx<T>{-c1, -sg * s1});
#pragma unroll
  for (int k2 = 0; k2 < 4; ++k2) {
    cpx<T> t[4] = {a[0][k2], a[1][k2], a[2][k2], a[3][k2]};
    dft_small<4, INV>(t);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) v[k2 + 4 * k1] = t[k1];
  }
}

// Forward radix-8 DFT -> low band of the default alpha = 0.5 at N = 2048
// (cutoff N/4: of the bins k = j + 256 r only r = 0, 1, 6, 7 survive, r = 6
// not at j = 0) -> inverse radix-8 DFT, without computing the masked outputs
// or multiplying by the zeroed inputs.  Same DFT definitions as dft_small<8>.
template <typename T>
__device__ __forceinline__ void lowband8_fwd_inv(cpx<T>* w, bool zero6) {
  const T h = (T)0.70710678118654752440;
  // forward, decimation in frequency: even outputs from a, odd from b
  const cpx<T> a0 = cadd(w[0], w[4]), a1 = cadd(w[1], w[5]);
  const cpx<T> a2 = cadd(w[2], w[6]), a3 = cadd(w[3], w[7]);
  const cpx<T> b0 = csub(w[0], w[4]);
  const cpx<T> b1 = cmul(csub(w[1], w[5]), cpx<T>{h, -h});
  const cpx<T> b2 = mul_mi<false>(csub(w[2], w[6]));
  const cpx<T> b3 = cmul(csub(w[3], w[7]), cpx<T>{-h, -h});
  const cpx<T> y0 = cadd(cadd(a0, a2), cadd(a1, a3));
  cpx<T> y6 = cadd(csub(a0, a2), mul_mi<true>(csub(a1, a3)));   // + i (a1 - a3)
  const cpx<T> y1 = cadd(cadd(b0, b2), cadd(b1, b3));
  const cpx<T> y7 = cadd(csub(b0, b2), mul_mi<true>(csub(b1, b3)));
  if (zero6) y6 = cpx<T>{(T)0, (T)0};
  // inverse from bins 0, 1, 6, 7: E_p = y0 + (-i)^p y6, O_p = y1 + (-i)^p y7
  const cpx<T> e0 = cadd(y0, y6), e2 = csub(y0, y6);
  const cpx<T> e1 = cadd(y0, mul_mi<false>(y6)), e3 = cadd(y0, mul_mi<true>(y6));
  const cpx<T> o0 = cadd(y1, y7), o2 = csub(y1, y7);
  const cpx<T> o1 = cmul(cadd(y1, mul_mi<false>(y7)), cpx<T>{h, h});
  const cpx<T> o3 = cmul(cadd(y1, mul_mi<true>(y7)), cpx<T>{-h, h});
  const cpx<T> o2i = mul_mi<true>(o2);
  w[0] = cadd(e0, o0);
  w[4] = csub(e0, o0);
  w[1] = cadd(e1, o1);
  w[5] = csub(e1, o1);
  w[2] = cadd(e2, o2i);
  w[6] = csub(e2, o2i);
  w[3] = cadd(e3, o3);
  w[7] = csub(e3, o3);
}

template <int R, bool INV, typename T>
__device__ __forceinline__ void dft_r(cpx<T>* v) {
  if constexpr (R == 16) dft16<INV>(v);
  else dft_small<R, INV>(v);
}

template <bool INV, typename T>
__device__ __forceinline__ cpx<T> twl(const cpx<T>* __restrict__ tw, int idx) {
  cpx<T> w = tw[idx];
  if (INV) w.y = -w.y;
  return w;
}

// v[r] *= W_N^{(a*r) mod N} (conjugated for INV), r = 1..R-1.
template <int R, bool INV, int N, typename T>
__device__ __forceinline__ void twiddle(cpx<T>* v, const cpx<T>* __restrict__ tw, int a) {
  if (a == 0) return;
  cpx<T> w[16];
  w[1] = twl<INV>(tw, a & (N - 1));
  if constexpr (R > 2) {
    w[2] = twl<INV>(tw, (2 * a) & (N - 1));
    w[3] = cmul(w[1], w[2]);
  }
  if constexpr (R > 4) {
    w[4] = twl<INV>(tw, (4 * a) & (N - 1));
    w[5] = cmul(w[1], w[4]);
    w[6] = cmul(w[2], w[4]);
    w[7] = cmul(w[3], w[4]);
  }
  if constexpr (R > 8) {
    w[8] = twl<INV>(tw, (8 * a) & (N - 1));
#pragma unroll
    for (int r = 9; r < 16; ++r) w[r] = cmul(w[r - 8], w[8]);
  }
#pragma unroll
  for (int r = 1; r < R; ++r) v[r] = cmul(v[r], w[r]);
}

// Exchange-buffer index.  16-B elements (f64 complex) are served 8 threads per
// shared-memory wavefront: an XOR of the low 3 index bits with bits 3-6 keeps
// every exchange pattern (stride 1, 16, R3 and the Stockham output scatter)
// conflict-free without padding.  8-B elements (f32 complex, 16 threads per
// wavefront) use one pad element per 16.
template <typename T>
__device__ __forceinline__ int sp16(int i) {
  if constexpr (sizeof(T) == 8) return i ^ (((i >> 3) ^ (i >> 4)) & 7);
  else return i + (i >> 4);
}

template <int GT>
__device__ __forceinline__ void group_sync(int g) {
  if constexpr (GT == 32) {
    __syncwarp();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "r"(GT) : "memory");
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <typename T, typename IN, int R3, int SPT = 1>
struct Fft2Cfg {
  static constexpr int THREADS = FFT2_THREADS / SPT;  // SPT signals per thread
  static constexpr int N = 256 * R3;
  static constexpr int GT = N / 16;                 // threads per signal group
  static constexpr int NG = THREADS / GT;           // groups per CTA
  static constexpr int NS = NG * SPT;               // signals per tile
  static constexpr int TW = 2 * NS;                 // lanes per tile
  static constexpr int SIGPAD = sizeof(T) == 8 ? N : N + N / 16;  // signal buffer (elements)
  static constexpr size_t SIG_BYTES = (size_t)NS * SIGPAD * sizeof(cpx<T>);
  static constexpr size_t TILE_BYTES = (size_t)N * TW * sizeof(IN);
  static constexpr size_t ACC_BYTES = (size_t)N * sizeof(double);
  // twiddle tables: f2 [16 r][16 (t&15)], i2 [16 r][R3 (t%R3)], and (when it
  // fits) the per-thread table T3 [16 r][GT t] = W_N^{t r} for f3 / i3
  // (+ 16 entries W_N^{q GT r} for the f3 twiddles of butterflies q > 0)
  static constexpr size_t T2_BYTES = (size_t)(16 * (16 + R3) + 16) * sizeof(cpx<T>);
  static constexpr size_t T3_BYTES = (size_t)16 * GT * sizeof(cpx<T>);
  static constexpr size_t BASE = SIG_BYTES + TILE_BYTES + ACC_BYTES + T2_BYTES;
  static constexpr bool USE_T3 = BASE + T3_BYTES <= 227 * 1024;
  static constexpr size_t SMEM = BASE + (USE_T3 ? T3_BYTES : 0);
  static_assert(NS * N == 8192, "8192 points in flight per CTA");
};

// Stage tile `it` (lanes lt0 .. lt0+TW) of rows [0, N) into smem.
template <typename IN, int N, int TW, int THREADS>
__device__ __forceinline__ void load_tile(IN* tile, const IN* base, int64_t ld_token, int lt0,
                                          int lane_end, bool vec_ok) {
  constexpr bool whole = (TW * sizeof(IN)) % 16 == 0;
  if constexpr (whole) {
    constexpr int CPR = TW * (int)sizeof(IN) / 16;  // 16-B chunks per row
    if (vec_ok && lt0 + TW <= lane_end) {
      for (int q = threadIdx.x; q < N * CPR; q += THREADS) {
        const int n = q / CPR, ch = q % CPR;
        cp_async16(reinterpret_cast<char*>(tile) + (size_t)q * 16,
                   reinterpret_cast<const char*>(base + (int64_t)n * ld_token + lt0) + ch * 16);
      }
      cp_async_commit();
      return;
    }
  }
  {
    for (int q = threadIdx.x; q < N * TW; q += THREADS) {
      const int n = q / TW, c = q % TW;
      const int lane = lt0 + c;
      tile[q] = lane < lane_end ? base[(int64_t)n * ld_token + lane] : IN(0.0f);
    }
  }
  cp_async_commit();
}

// LB: the default band (alpha = 0.5 at N = 2048, cutoff N/4) with the pruned
// radix-8 middle passes (lowband8_fwd_inv).
template <typename T, typename IN, int R3, int SPT, bool LB = false>
__global__ void __launch_bounds__(FFT2_THREADS / SPT, 1)
fft2_energy_kernel(const IN* __restrict__ keys, const IN* __restrict__ values, int L, int lanes,
                   int64_t ld_token, int64_t ld_layer, int64_t ld_chunk, int cutoff,
                   const cpx<T>* __restrict__ tw, double* __restrict__ partial) {
  using Cfg = Fft2Cfg<T, IN, R3, SPT>;
  constexpr int N = Cfg::N, GT = Cfg::GT, TW = Cfg::TW, THREADS = Cfg::THREADS;
  constexpr int Q = 16 / R3;          // radix-R3 butterflies per thread
  constexpr int NR3 = N / R3;         // = 256
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cpx<T>* sigall = reinterpret_cast<cpx<T>*>(smem_raw);
  IN* tile = reinterpret_cast<IN*>(smem_raw + Cfg::SIG_BYTES);
  // per-token energy of the CTA's signals, summed signal by signal in a fixed
  // order (registers hold the FFT; a per-thread f64 accumulator would spill)
  double* acc = reinterpret_cast<double*>(smem_raw + Cfg::SIG_BYTES + Cfg::TILE_BYTES);
  cpx<T>* t2f = reinterpret_cast<cpx<T>*>(smem_raw + Cfg::SIG_BYTES + Cfg::TILE_BYTES +
                                          Cfg::ACC_BYTES);
  cpx<T>* t2i = t2f + 16 * 16;
  cpx<T>* tq = t2i + 16 * R3;  // [Q][R3] W_N^{q GT r}
  cpx<T>* t3 = tq + 16;
  // tables from the N-point table (exact entries: no products)
  for (int q = threadIdx.x; q < 16 * 16; q += THREADS) {
    const int r = q / 16, u = q % 16;
    t2f[q] = tw[(u * r * R3) & (N - 1)];
  }
  for (int q = threadIdx.x; q < 16 * R3; q += THREADS) {
    const int r = q / R3, u = q % R3;
    cpx<T> w = tw[(u * r * 16) & (N - 1)];
    w.y = -w.y;
    t2i[q] = w;
  }
  for (int q = threadIdx.x; q < Q * R3; q += THREADS) {
    const int qq = q / R3, r = q % R3;
    tq[q] = tw[(qq * GT * r) & (N - 1)];
  }
  if constexpr (Cfg::USE_T3) {
    for (int q = threadIdx.x; q < 16 * GT; q += THREADS) {
      const int r = q / GT, u = q % GT;
      t3[q] = tw[(u * r) & (N - 1)];
    }
  }

  // group g owns signals g*SPT .. g*SPT+SPT-1 of every tile (lanes 2 sig, 2 sig + 1)
  const int g = threadIdx.x / GT, t = threadIdx.x % GT;
  cpx<T>* sigs[SPT];
#pragma unroll
  for (int s = 0; s < SPT; ++s) sigs[s] = sigall + (g * SPT + s) * Cfg::SIGPAD;
  const int lb = blockIdx.x, tensor = blockIdx.y;
  const int c = blockIdx.z / L, l = blockIdx.z % L;
  const IN* base = (tensor == 0 ? keys : values) + (int64_t)c * ld_chunk + (int64_t)l * ld_layer;
  const int lane0 = lb * LANE_BLOCK;
  const int lane_end = min(lanes, lane0 + LANE_BLOCK);
  const int iters = (lane_end - lane0 + TW - 1) / TW;
  const bool vec_ok = ((ld_token * (int64_t)sizeof(IN)) % 16 == 0) &&
                      (((uintptr_t)base) % 16 == 0) && ((lane0 * (int)sizeof(IN)) % 16 == 0);

  for (int n = threadIdx.x; n < N; n += THREADS) acc[n] = 0.0;
  load_tile<IN, N, TW, THREADS>(tile, base, ld_token, lane0, lane_end, vec_ok);
  cp_async_wait_all();
  __syncthreads();
  // per-thread energies of tokens t + GT r over this thread's signals, in a
  // fixed order (its signals, tile by tile); the groups are merged once at
  // the end in group order
  double eacc[16];
#pragma unroll
  for (int r = 0; r < 16; ++r) eacc[r] = 0.0;
  for (int it = 0; it < iters; ++it) {
    cpx<T> v[SPT][16];
    // f1 input: lanes (2 sig, 2 sig + 1) of tokens t + GT r
#pragma unroll
    for (int s = 0; s < SPT; ++s) {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        const IN* p = tile + (size_t)(t + GT * r) * TW + 2 * (g * SPT + s);
        v[s][r] = {(T)to_f32(p[0]), (T)to_f32(p[1])};
      }
    }
    __syncthreads();
    if (it + 1 < iters)
      load_tile<IN, N, TW, THREADS>(tile, base, ld_token, lane0 + (it + 1) * TW, lane_end, vec_ok);

    // ---- forward f1: radix 16, Ns = 1
#pragma unroll
    for (int s = 0; s < SPT; ++s) dft16<false>(v[s]);
    group_sync<GT>(g);  // previous signal's i3 reads of sig are done
#pragma unroll
    for (int s = 0; s < SPT; ++s)
#pragma unroll
      for (int r = 0; r < 16; ++r) sigs[s][sp16<T>(16 * t + r)] = v[s][r];
    group_sync<GT>(g);
    // ---- f2: radix 16, Ns = 16
#pragma unroll
    for (int s = 0; s < SPT; ++s) {
#pragma unroll
      for (int r = 0; r < 16; ++r) v[s][r] = sigs[s][sp16<T>(t + GT * r)];
#pragma unroll
      for (int r = 1; r < 16; ++r) v[s][r] = cmul(v[s][r], t2f[r * 16 + (t & 15)]);
      dft16<false>(v[s]);
    }
    group_sync<GT>(g);
#pragma unroll
    for (int s = 0; s < SPT; ++s)
#pragma unroll
      for (int r = 0; r < 16; ++r) sigs[s][sp16<T>((t >> 4) * 256 + (t & 15) + 16 * r)] = v[s][r];
    group_sync<GT>(g);
    // ---- f3: radix R3, Ns = N/R3; mask; i1: inverse radix R3, Ns = 1
#pragma unroll
    for (int s = 0; s < SPT; ++s) {
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int j = t + q * GT;
        cpx<T>* w = v[s] + q * R3;
#pragma unroll
        for (int r = 0; r < R3; ++r) w[r] = sigs[s][sp16<T>(j + NR3 * r)];
        if constexpr (Cfg::USE_T3) {
          // W_N^{(t + q GT) r} = W_N^{t r} W_N^{q GT r}
#pragma unroll
          for (int r = 1; r < R3; ++r) {
            cpx<T> tr = t3[r * GT + t];
            if (q > 0) tr = cmul(tr, tq[q * R3 + r]);
            w[r] = cmul(w[r], tr);
          }
        } else {
          twiddle<R3, false, N>(w, tw, j);
        }
        if constexpr (LB && R3 == 8) {
          lowband8_fwd_inv(w, j == 0);
        } else {
          dft_r<R3, false>(w);
#pragma unroll
          for (int r = 0; r < R3; ++r) {
            const int k = j + NR3 * r;
            const int kk = k < N - k ? k : N - k;
            if (cutoff >= 0 ? kk >= cutoff : kk < -cutoff - 1) w[r] = {(T)0, (T)0};
          }
          dft_r<R3, true>(w);
        }
      }
    }
    group_sync<GT>(g);
#pragma unroll
    for (int s = 0; s < SPT; ++s)
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int j = t + q * GT;
#pragma unroll
        for (int r = 0; r < R3; ++r) sigs[s][sp16<T>(j * R3 + r)] = v[s][q * R3 + r];
      }
    group_sync<GT>(g);
    // ---- i2: inverse radix 16, Ns = R3
#pragma unroll
    for (int s = 0; s < SPT; ++s) {
#pragma unroll
      for (int r = 0; r < 16; ++r) v[s][r] = sigs[s][sp16<T>(t + GT * r)];
#pragma unroll
      for (int r = 1; r < 16; ++r) v[s][r] = cmul(v[s][r], t2i[r * R3 + (t % R3)]);
      dft16<true>(v[s]);
    }
    group_sync<GT>(g);
#pragma unroll
    for (int s = 0; s < SPT; ++s)
#pragma unroll
      for (int r = 0; r < 16; ++r)
        sigs[s][sp16<T>((t / R3) * (16 * R3) + (t % R3) + R3 * r)] = v[s][r];
    group_sync<GT>(g);
    // ---- i3: inverse radix 16, Ns = N/16 -> token t + GT r in v[r]
#pragma unroll
    for (int s = 0; s < SPT; ++s) {
#pragma unroll
      for (int r = 0; r < 16; ++r) v[s][r] = sigs[s][sp16<T>(t + GT * r)];
      if constexpr (Cfg::USE_T3) {
#pragma unroll
        for (int r = 1; r < 16; ++r) {
          cpx<T> w = t3[r * GT + t];
          w.y = -w.y;
          v[s][r] = cmul(v[s][r], w);
        }
      } else {
        twiddle<16, true, N>(v[s], tw, t);
      }
      dft16<true>(v[s]);
    }
#pragma unroll
    for (int s = 0; s < SPT; ++s)
#pragma unroll
      for (int r = 0; r < 16; ++r)
        eacc[r] += (double)(v[s][r].x * v[s][r].x + v[s][r].y * v[s][r].y);
    cp_async_wait_all();  // next tile landed; the barrier publishes it (and frees sig)
    __syncthreads();
  }
  // merge the groups' energies in group order (deterministic)
  for (int gg = 0; gg < Cfg::NG; ++gg) {
    if (g == gg) {
#pragma unroll
      for (int r = 0; r < 16; ++r) acc[t + GT * r] += eacc[r];
    }
    __syncthreads();
  }
  const double inv_n2 = 1.0 / ((double)N * (double)N);
  const int nlb = gridDim.x;
  double* out = partial + ((((int64_t)blockIdx.z * 2 + tensor) * nlb) + lb) * N;
  for (int n = threadIdx.x; n < N; n += THREADS) out[n] = acc[n] * inv_n2;
}

// ---------------------------------------------------------------------------
// Mixed-radix path for smooth lengths N = 2^a 3^b 5^c 7^d (e.g. 96, 1000, 1536,
// 3000) that are not powers of two: the same forward FFT -> band mask ->
// inverse FFT -> |recon|^2 as above, Stockham passes of radix 8/4/2/3/5/7
// chosen at run time, ping-pong shared-memory buffers (one barrier per pass).
// N with a prime factor > 7 keeps the direct circulant path.
// ---------------------------------------------------------------------------
constexpr int MR_THREADS = 512;
constexpr int MR_MAX_N = 5120;  // f64: 2 x 5120 x 16 B buffers + 40 KB energies
constexpr int MR_MAX_PASSES = 16;

struct MrPlan {
  int n_pass;
  int radix[MR_MAX_PASSES];
};

// W_R^m = (cos 2 pi m / R, sin 2 pi m / R), correctly rounded, m = 0..R-1
__constant__ double c_cos3[3] = {1.0, -0.5, -0.5};
__constant__ double c_sin3[3] = {0.0, 0.8660254037844386, -0.8660254037844386};
__constant__ double c_cos5[5] = {1.0, 0.30901699437494745, -0.8090169943749475, -0.8090169943749475,
                                 0.30901699437494745};
__constant__ double c_sin5[5] = {0.0, 0.9510565162951535, 0.5877852522924731, -0.5877852522924731,
                                 -0.9510565162951535};
__constant__ double c_cos7[7] = {1.0, 0.6234898018587335, -0.2225209339563144, -0.9009688679024191,
                                 -0.9009688679024191, -0.2225209339563144, 0.6234898018587335};
__constant__ double c_sin7[7] = {0.0, 0.7818314824680298, 0.9749279121818236, 0.4338837391175581,
                                 -0.4338837391175581, -0.9749279121818236, -0.7818314824680298};

// y[k] = sum_n x[n] W_R^{-+nk} for a small prime R (forward sign -, inverse +)
template <int R, bool INV, typename T>
__device__ __forceinline__ void dft_prime(cpx<T>* v) {
  const double* cs = R == 3 ? c_cos3 : R == 5 ? c_cos5 : c_cos7;
  const double* sn = R == 3 ? c_sin3 : R == 5 ? c_sin5 : c_sin7;
  cpx<T> y[R];
#pragma unroll
  for (int k = 0; k < R; ++k) {
    cpx<T> acc = v[0];
#pragma unroll
    for (int n = 1; n < R; ++n) {
      const int m = (n * k) % R;
      const T c = (T)cs[m], sv = INV ? (T)sn[m] : (T)-sn[m];
      acc.x += v[n].x * c - v[n].y * sv;
      acc.y += v[n].x * sv + v[n].y * c;
    }
    y[k] = acc;
  }
#pragma unroll
  for (int k = 0; k < R; ++k) v[k] = y[k];
}

template <int R, bool INV, typename T>
__device__ __forceinline__ void dft_any(cpx<T>* v) {
  if constexpr (R == 2 || R == 4 || R == 8) dft_small<R, INV>(v);
  else dft_prime<R, INV>(v);
}

// One Stockham pass (radix R, Ns = product of the earlier radices) from `in`
// to `out` over S signals.  MASK zeroes the band-rejected bins on load (first
// inverse pass); ENERGY stores |z|^2 in .x (last inverse pass).
template <int R, bool INV, typename T>
__device__ __forceinline__ void mr_pass(const cpx<T>* in, cpx<T>* out, int S, int N, int Ns,
                                        const cpx<T>* __restrict__ tw, bool mask, int cutoff,
                                        bool energy) {
  const int NB = N / R;
  const int step = N / (Ns * R);
  for (int b = threadIdx.x; b < S * NB; b += MR_THREADS) {
    const int sg = b / NB, j = b - sg * NB;
    const int jm = j % Ns;
    cpx<T> v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int idx = j + r * NB;
      cpx<T> val = in[sg * N + idx];
      if (mask) {
        const int kk = idx < N - idx ? idx : N - idx;
        if (cutoff >= 0 ? kk >= cutoff : kk < -cutoff - 1) val = {(T)0, (T)0};
      }
      if (r > 0 && jm > 0) {
        // jm * step * r < (N / R) * R = N: no modular reduction needed
        cpx<T> w = tw[jm * step * r];
        if (INV) w.y = -w.y;
        val = cmul(val, w);
      }
      v[r] = val;
    }
    dft_any<R, INV>(v);
    const int base = (j / Ns) * Ns * R + jm;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (energy) out[sg * N + base + r * Ns] = {v[r].x * v[r].x + v[r].y * v[r].y, (T)0};
      else out[sg * N + base + r * Ns] = v[r];
    }
  }
}

template <bool INV, typename T>
__device__ __forceinline__ void mr_pass_any(int R, const cpx<T>* in, cpx<T>* out, int S, int N,
                                            int Ns, const cpx<T>* tw, bool mask, int cutoff,
                                            bool energy) {
  switch (R) {
    case 8: mr_pass<8, INV>(in, out, S, N, Ns, tw, mask, cutoff, energy); break;
    case 4: mr_pass<4, INV>(in, out, S, N, Ns, tw, mask, cutoff, energy); break;
    case 2: mr_pass<2, INV>(in, out, S, N, Ns, tw, mask, cutoff, energy); break;
    case 3: mr_pass<3, INV>(in, out, S, N, Ns, tw, mask, cutoff, energy); break;
    case 5: mr_pass<5, INV>(in, out, S, N, Ns, tw, mask, cutoff, energy); break;
    default: mr_pass<7, INV>(in, out, S, N, Ns, tw, mask, cutoff, energy); break;
  }
}

// grid: x = lane block, y = tensor, z = c*L + l; S signals (2S lanes) in
// flight per CTA, as many as the ping-pong buffers leave room for.
template <typename T, typename IN>
__global__ void __launch_bounds__(MR_THREADS, 1)
fftmr_energy_kernel(const IN* __restrict__ keys, const IN* __restrict__ values, int N, int L,
                    int lanes, int64_t ld_token, int64_t ld_layer, int64_t ld_chunk, int cutoff,
                    const cpx<T>* __restrict__ tw, MrPlan plan, int S,
                    double* __restrict__ partial) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cpx<T>* buf0 = reinterpret_cast<cpx<T>*>(smem_raw);
  cpx<T>* buf1 = buf0 + S * N;
  double* acc = reinterpret_cast<double*>(buf1 + S * N);
  const int lb = blockIdx.x, tensor = blockIdx.y;
  const int c = blockIdx.z / L, l = blockIdx.z % L;
  const IN* base = (tensor == 0 ? keys : values) + (int64_t)c * ld_chunk + (int64_t)l * ld_layer;
  const int lane0 = lb * LANE_BLOCK, lane_end = min(lanes, lane0 + LANE_BLOCK);
  for (int n = threadIdx.x; n < N; n += MR_THREADS) acc[n] = 0.0;
  for (int g0 = lane0; g0 < lane_end; g0 += 2 * S) {
    for (int q = threadIdx.x; q < S * N; q += MR_THREADS) {
      const int sg = q / N, n = q - sg * N;
      const int la = g0 + 2 * sg, lbn = la + 1;
      const IN* row = base + (int64_t)n * ld_token;
      buf0[q] = {la < lane_end ? (T)load_as_double(row + la) : (T)0,
                 lbn < lane_end ? (T)load_as_double(row + lbn) : (T)0};
    }
    __syncthreads();
    cpx<T>* src = buf0;
    cpx<T>* dst = buf1;
    int Ns = 1;
    for (int p = 0; p < plan.n_pass; ++p) {  // forward
      mr_pass_any<false>(plan.radix[p], src, dst, S, N, Ns, tw, false, cutoff, false);
      Ns *= plan.radix[p];
      __syncthreads();
      cpx<T>* t = src; src = dst; dst = t;
    }
    Ns = 1;
    for (int p = 0; p < plan.n_pass; ++p) {  // inverse, mask on the first pass
      mr_pass_any<true>(plan.radix[p], src, dst, S, N, Ns, tw, p == 0, cutoff,
                        p == plan.n_pass - 1);
      Ns *= plan.radix[p];
      __syncthreads();
      cpx<T>* t = src; src = dst; dst = t;
    }
    // energies in src[sg][n].x: fixed-order sum over the group's signals
    for (int n = threadIdx.x; n < N; n += MR_THREADS) {
      double e = 0.0;
      for (int sg = 0; sg < S; ++sg) e += (double)src[sg * N + n].x;
      acc[n] += e;
    }
    __syncthreads();
  }
  const double inv_n2 = 1.0 / ((double)N * (double)N);
  const int nlb = gridDim.x;
  double* out = partial + ((((int64_t)blockIdx.z * 2 + tensor) * nlb) + lb) * N;
  for (int n = threadIdx.x; n < N; n += MR_THREADS) out[n] = acc[n] * inv_n2;
}

static bool mr_plan(int64_t N, MrPlan* plan) {
  if (N < 2 || N > MR_MAX_N) return false;
  int64_t m = N;
  plan->n_pass = 0;
  const int order[6] = {8, 4, 2, 3, 5, 7};
  for (int i = 0; i < 6; ++i) {
    const int r = order[i];
    while (m % r == 0) {
      if (plan->n_pass == MR_MAX_PASSES) return false;
      plan->radix[plan->n_pass++] = r;
      m /= r;
    }
  }
  return m == 1;
}

template <typename T>
static int mr_signals(int64_t N) {
  const int64_t room = 227 * 1024 - N * (int64_t)sizeof(double);
  int64_t S = room / (2 * N * (int64_t)sizeof(cpx<T>));
  if (S > 64) S = 64;  // 128-lane blocks
  return (int)(S < 1 ? 1 : S);
}

template <typename T>
static size_t mr_smem(int64_t N) {
  return (size_t)(2 * mr_signals<T>(N) * N) * sizeof(cpx<T>) + (size_t)N * sizeof(double);
}

template <typename T, typename IN>
static int launch_mr(const void* k, const void* v, int64_t N, int L, int C, int lanes, int64_t ldt,
                     int64_t ldl, int64_t ldc, int cutoff, const void* tw, const MrPlan& plan,
                     double* partial, cudaStream_t st) {
  auto kern = fftmr_energy_kernel<T, IN>;
  const size_t smem = mr_smem<T>(N);
  CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int nlb = (lanes + LANE_BLOCK - 1) / LANE_BLOCK;
  dim3 grid(nlb, 2, C * L);
  kern<<<grid, MR_THREADS, smem, st>>>((const IN*)k, (const IN*)v, (int)N, L, lanes, ldt, ldl, ldc,
                                       cutoff, (const cpx<T>*)tw, plan, mr_signals<T>(N), partial);
  return check_launch("fftmr_energy_kernel");
}

// Circulant band kernel p[m] = (1/N) sum_{k in band} w_k cos(2 pi k m/N) over
// rfft bins k in [0, N/2] (w_k = 1 for DC and an even-N Nyquist bin, else 2):
// the exact impulse response of rfft -> zero the other bins -> irfft.  Low band
// (cutoff = c >= 0) keeps k < c; cutoff = -(c+1) keeps the high band k >= c.
// An empty band sums nothing, so its scores are exactly 0 like the reference's.
__global__ void lowpass_kernel_table(int N, int cutoff, double* p) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= N) return;
  const bool high = cutoff < 0;
  const int c = high ? -cutoff - 1 : cutoff;
  const int klo = high ? c : 0;
  const int khi = high ? N / 2 : min(c - 1, N / 2);
  double s = 0.0;
  for (int k = klo; k <= khi; ++k) {
    const long long km = ((long long)k * m) % N;
    const double w = (k == 0 || 2 * k == N) ? 1.0 : 2.0;
    s += w * cospi(2.0 * (double)km / (double)N);
  }
  p[m] = s / (double)N;
}

__global__ void twiddle_table(int N, cpx<double>* twd, cpx<float>* twf) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= N) return;
  double s, c;
  sincospi(2.0 * (double)m / (double)N, &s, &c);
  if (twd) twd[m] = {c, -s};
  if (twf) twf[m] = {(float)c, (float)-s};
}

// Direct path: y[i][lane] = sum_j p[(i-j) mod N] x[j][lane]; energy per token.
// grid: x = token tile (32 tokens), y = tensor*nlb + lane block, z = c*L + l.
template <typename IN>
__global__ void __launch_bounds__(256)
direct_energy_kernel(const IN* __restrict__ keys, const IN* __restrict__ values,
                     int N, int L, int lanes, int64_t ld_token, int64_t ld_layer,
                     int64_t ld_chunk, const double* __restrict__ p, int nlb,
                     double* __restrict__ partial) {
  const int tensor = blockIdx.y / nlb, lb = blockIdx.y % nlb;
  const int c = blockIdx.z / L, l = blockIdx.z % L;
  const IN* base = (tensor == 0 ? keys : values) + (int64_t)c * ld_chunk + (int64_t)l * ld_layer;
  const int lane0 = lb * LANE_BLOCK, lane_end = min(lanes, lane0 + LANE_BLOCK);
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // 8 warps x 4 tokens
  __shared__ double red[8][4][33];
  double energy[4] = {0, 0, 0, 0};
  const int i0 = blockIdx.x * 32 + ty * 4;
  for (int ls = lane0; ls < lane_end; ls += 32) {
    const int lane = ls + tx;
    double y[4] = {0, 0, 0, 0};
    if (lane < lane_end) {
      for (int j = 0; j < N; ++j) {
        const double xv = load_as_double(base + (int64_t)j * ld_token + lane);
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int i = i0 + t;
          if (i < N) {
            int m = i - j;
            m += (m < 0) ? N : 0;
            y[t] += p[m] * xv;
          }
        }
      }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) energy[t] += y[t] * y[t];
  }
  // fixed-order reduction over the 32 lanes of the warp
#pragma unroll
  for (int t = 0; t < 4; ++t) red[ty][t][tx] = energy[t];
  __syncwarp();
  if (tx < 4) {
    double e = 0.0;
    for (int q = 0; q < 32; ++q) e += red[ty][tx][q];
    const int i = i0 + tx;
    if (i < N)
      partial[((((int64_t)blockIdx.z * 2 + tensor) * nlb) + lb) * N + i] = e;
  }
}

// Per (chunk, token): layer score = 0.5*sqrt(EK) + 0.5*sqrt(EV); aggregate =
// sequential layer sum / L (ct/spectral.py:74-78, :156).
__global__ void combine_scores(const double* __restrict__ partial, int C, int L, int N,
                               int nlb, double* __restrict__ layer_scores,
                               double* __restrict__ agg) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)C * N) return;
  const int c = (int)(t / N), n = (int)(t % N);
  double total = 0.0;
  for (int l = 0; l < L; ++l) {
    double e[2];
    for (int tensor = 0; tensor < 2; ++tensor) {
      const double* src = partial + ((((int64_t)(c * L + l) * 2 + tensor) * nlb) * N) + n;
      double s = 0.0;
      for (int b = 0; b < nlb; ++b) s += src[(int64_t)b * N];
      e[tensor] = s;
    }
    double score = 0.0;
    score += 0.5 * sqrt(e[0]);
    score += 0.5 * sqrt(e[1]);
    layer_scores[((int64_t)c * L + l) * N + n] = score;
    total += score;
  }
  if (agg) agg[t] = total / (double)L;
}

// Block bitonic sort of one row: descending score, ascending index on ties.
constexpr int SORT_THREADS = 1024;
__global__ void __launch_bounds__(SORT_THREADS)
desc_order_kernel(const double* __restrict__ scores, int n, int P, int32_t* __restrict__ order) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* key = reinterpret_cast<double*>(smem_raw);
  int* idx = reinterpret_cast<int*>(key + P);
  const double* row = scores + (int64_t)blockIdx.x * n;
  for (int i = threadIdx.x; i < P; i += SORT_THREADS) {
    key[i] = i < n ? row[i] : -INFINITY;
    idx[i] = i < n ? i : 0x7fffffff;
  }
  __syncthreads();
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += SORT_THREADS) {
        const int ixj = i ^ j;
        if (ixj > i) {
          const double ka = key[i], kb = key[ixj];
          const int ia = idx[i], ib = idx[ixj];
          // before(x, y): x.score > y.score || (== && x.idx < y.idx)
          const bool b_before_a = (kb > ka) || (kb == ka && ib < ia);
          const bool a_before_b = (ka > kb) || (ka == kb && ia < ib);
          const bool asc = ((i & k) == 0);
          if (asc ? b_before_a : a_before_b) {
            key[i] = kb; key[ixj] = ka;
            idx[i] = ib; idx[ixj] = ia;
          }
        }
      }
      __syncthreads();
    }
  }
  int32_t* out = order + (int64_t)blockIdx.x * n;
  for (int i = threadIdx.x; i < n; i += SORT_THREADS) out[i] = idx[i];
}

// Selection plan: one CTA per chunk.  Marks the first k entries of the
// aggregate order, then emits recomputed / kept tokens in ascending order
// (ct/spectral.py:175-184) on the global axis (offset by the chunk start).
constexpr int PLAN_THREADS = 1024;
// One chunk's plan: tokens [off, off + n) with aggregate order agg[0..n); the
// first k ranks are recomputed.  rec / keep ascending, ksrc = rank of each
// keep token (nullable).  rank[] = n ints of shared memory.
__device__ __forceinline__ void plan_one(const int32_t* __restrict__ agg, int64_t off, int n,
                                         int k, int* rank, int* warp_tot, int32_t* rec,
                                         int32_t* keep, int32_t* ksrc) {
  for (int i = threadIdx.x; i < n; i += PLAN_THREADS) rank[agg[i]] = i;
  __syncthreads();
  // contiguous segment per thread
  const int per = (n + PLAN_THREADS - 1) / PLAN_THREADS;
  const int t0 = min(n, (int)threadIdx.x * per), t1 = min(n, t0 + per);
  int cnt = 0;
  for (int t = t0; t < t1; ++t) cnt += rank[t] < k;
  // block exclusive scan of cnt
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = cnt;
  for (int d = 1; d < 32; d <<= 1) {
    int v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = lane < PLAN_THREADS / 32 ? warp_tot[lane] : 0;
    int wi = w;
    for (int d = 1; d < 32; d <<= 1) {
      int v = __shfl_up_sync(0xffffffffu, wi, d);
      if (lane >= d) wi += v;
    }
    if (lane < PLAN_THREADS / 32) warp_tot[lane] = wi - w;
  }
  __syncthreads();
  int rpos = warp_tot[warp] + incl - cnt;  // recomputed tokens before my segment
  int kpos = t0 - rpos;                    // kept tokens before my segment
  for (int t = t0; t < t1; ++t) {
    const int rk = rank[t];
    if (rk < k) {
      rec[rpos++] = (int32_t)(off + t);
    } else {
      if (ksrc) ksrc[kpos] = rk;
      keep[kpos++] = (int32_t)(off + t);
    }
  }
}

__global__ void __launch_bounds__(PLAN_THREADS)
selection_plan_kernel(const int32_t* __restrict__ agg_orders, const int64_t* __restrict__ offsets,
                      const int64_t* __restrict__ ks, const int64_t* __restrict__ rec_base,
                      const int64_t* __restrict__ keep_base, int32_t* __restrict__ rec_global,
                      int32_t* __restrict__ keep_global, int32_t* __restrict__ keep_src_row) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int warp_tot[PLAN_THREADS / 32];
  const int c = blockIdx.x;
  const int64_t off = offsets[c];
  plan_one(agg_orders + off, off, (int)(offsets[c + 1] - off), (int)ks[c],
           reinterpret_cast<int*>(smem_raw), warp_tot, rec_global + rec_base[c],
           keep_global + keep_base[c], keep_src_row ? keep_src_row + keep_base[c] : nullptr);
}

// ct_select: one chunk, scalar k (chunk-local token ids)
__global__ void __launch_bounds__(PLAN_THREADS)
select_kernel(const int32_t* __restrict__ order, int n, int k, int32_t* __restrict__ sel,
              int32_t* __restrict__ keep) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int warp_tot[PLAN_THREADS / 32];
  plan_one(order, 0, n, k, reinterpret_cast<int*>(smem_raw), warp_tot, sel, keep, nullptr);
}

static int ilog2_exact(int64_t n) {
  if (n <= 0 || (n & (n - 1))) return -1;
  int l = 0;
  while ((1LL << l) < n) ++l;
  return l;
}

static bool fft_path(int64_t N) {
  const int lg = ilog2_exact(N);
  return lg >= 3 && lg <= 13;
}

template <typename T, typename IN, int LOGN>
static int launch_fft_t(const void* k, const void* v, int L, int C, int lanes, int64_t ldt,
                        int64_t ldl, int64_t ldc, int cutoff, const void* tw,
                        double* partial, cudaStream_t st) {
  constexpr int N = 1 << LOGN;
  constexpr int PTS = ScoreCfg<T>::POINTS;
  constexpr int S = PTS / N < 1 ? 1 : (PTS / N > 64 ? 64 : PTS / N);
  const size_t smem = (size_t)(S * N + S * N / 8 + 8) * sizeof(cpx<T>);  // padded (spad)
  auto kern = fft_energy_kernel<T, IN, LOGN>;
  CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int nlb = (lanes + LANE_BLOCK - 1) / LANE_BLOCK;
  dim3 grid(nlb, 2, C * L);
  kern<<<grid, SCORE_THREADS, smem, st>>>((const IN*)k, (const IN*)v, L, lanes, ldt, ldl, ldc,
                                          cutoff, (const cpx<T>*)tw, partial);
  return check_launch("fft_energy_kernel");
}

// N = 2048: two signals per thread (8 warps, 254 registers) measured 4 % (f64) /
// 7 % (f32) faster than one signal per thread (16 warps, 128 registers)
static int g_fft2_spt = getenv("CT_SCORER_SPT") ? atoi(getenv("CT_SCORER_SPT")) : 2;
// CT_SCORER_NO_LB=1: generic masked middle passes even for the default band
static bool g_fft2_no_lb = getenv("CT_SCORER_NO_LB") != nullptr;

template <typename T, typename IN, int R3, int SPT, bool LB = false>
static int launch_fft2_spt(const void* k, const void* v, int L, int C, int lanes, int64_t ldt,
                           int64_t ldl, int64_t ldc, int cutoff, const void* tw, double* partial,
                           cudaStream_t st) {
  using Cfg = Fft2Cfg<T, IN, R3, SPT>;
  auto kern = fft2_energy_kernel<T, IN, R3, SPT, LB>;
  CT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
  const int nlb = (lanes + LANE_BLOCK - 1) / LANE_BLOCK;
  dim3 grid(nlb, 2, C * L);
  kern<<<grid, Cfg::THREADS, Cfg::SMEM, st>>>((const IN*)k, (const IN*)v, L, lanes, ldt, ldl, ldc,
                                              cutoff, (const cpx<T>*)tw, partial);
  return check_launch("fft2_energy_kernel");
}

template <typename T, typename IN, int R3>
static int launch_fft2_t(const void* k, const void* v, int L, int C, int lanes, int64_t ldt,
                         int64_t ldl, int64_t ldc, int cutoff, const void* tw, double* partial,
                         cudaStream_t st) {
  if (R3 == 8 && g_fft2_spt == 2) {
    if (cutoff == 256 * R3 / 4 && !g_fft2_no_lb)
      return launch_fft2_spt<T, IN, R3, 2, true>(k, v, L, C, lanes, ldt, ldl, ldc, cutoff, tw,
                                                 partial, st);
    return launch_fft2_spt<T, IN, R3, 2>(k, v, L, C, lanes, ldt, ldl, ldc, cutoff, tw, partial, st);
  }
  return launch_fft2_spt<T, IN, R3, 1>(k, v, L, C, lanes, ldt, ldl, ldc, cutoff, tw, partial, st);
}

static bool g_fft_v1_only = getenv("CT_SCORER_V1") != nullptr;

template <typename T, typename IN>
static int launch_fft(int logn, const void* k, const void* v, int L, int C, int lanes,
                      int64_t ldt, int64_t ldl, int64_t ldc, int cutoff, const void* tw,
                      double* partial, cudaStream_t st) {
  if (!g_fft_v1_only) {
    switch (logn) {
      case 9: return launch_fft2_t<T, IN, 2>(k, v, L, C, lanes, ldt, ldl, ldc, cutoff, tw, partial, st);
      case 10: return launch_fft2_t<T, IN, 4>(k, v, L, C, lanes, ldt, ldl, ldc, cutoff, tw, partial, st);
      case 11: return launch_fft2_t<T, IN, 8>(k, v, L, C, lanes, ldt, ldl, ldc, cutoff, tw, partial, st);
      case 12:  // f64 with f32 inputs does not fit one CTA at N = 4096: v1 below
        if (Fft2Cfg<T, IN, 16, 1>::SMEM <= 227 * 1024)
          return launch_fft2_t<T, IN, 16>(k, v, L, C, lanes, ldt, ldl, ldc, cutoff, tw, partial, st);
        break;
      default: break;
    }
  }
  switch (logn) {
#define CT_CASE(LG) \
  case LG: return launch_fft_t<T, IN, LG>(k, v, L, C, lanes, ldt, ldl, ldc, cutoff, tw, partial, st);
    CT_CASE(3) CT_CASE(4) CT_CASE(5) CT_CASE(6) CT_CASE(7) CT_CASE(8) CT_CASE(9)
    CT_CASE(10) CT_CASE(11) CT_CASE(12) CT_CASE(13)
#undef CT_CASE
    default: return fail(CT_ERR_UNSUPPORTED, "fft length 2^%d", logn);
  }
}

}  // namespace ct

using namespace ct;

extern "C" size_t ct_score_workspace_bytes(int64_t C, int64_t L, int64_t N, int64_t lanes,
                                           int precision) {
  (void)precision;
  const int64_t nlb = (lanes + LANE_BLOCK - 1) / LANE_BLOCK;
  size_t b = align_up((size_t)C * L * 2 * nlb * N * sizeof(double), 256);
  b += align_up((size_t)N * sizeof(cpx<double>), 256);  // twiddles / circulant
  b += align_up((size_t)N * sizeof(cpx<float>), 256);
  return b;
}

extern "C" int ct_desc_order(const double* scores, int64_t rows, int64_t n, int32_t* order,
                             void* stream) {
  if (rows < 0 || n < 0) return fail(CT_ERR_SHAPE, "negative sizes");
  if (rows == 0 || n == 0) return CT_OK;
  int64_t P = 1;
  while (P < n) P <<= 1;
  const size_t smem = (size_t)P * (sizeof(double) + sizeof(int));
  if (smem > 200 * 1024) return fail(CT_ERR_UNSUPPORTED, "order of %lld tokens exceeds one CTA", (long long)n);
  CT_CUDA(cudaFuncSetAttribute(desc_order_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  desc_order_kernel<<<(unsigned)rows, SORT_THREADS, smem, (cudaStream_t)stream>>>(scores, (int)n, (int)P, order);
  return check_launch("desc_order_kernel");
}

extern "C" int ct_score_chunks(const void* keys, const void* values, int dtype, int64_t C,
                               int64_t L, int64_t N, int64_t lanes, int64_t ld_token,
                               int64_t ld_layer, int64_t ld_chunk, int64_t cutoff, int precision,
                               double* layer_scores, double* agg_scores, int32_t* layer_order,
                               int32_t* agg_order, void* workspace, size_t workspace_bytes,
                               void* stream) {
  return ct_score_chunks_band(keys, values, dtype, C, L, N, lanes, ld_token, ld_layer, ld_chunk,
                              cutoff, precision, 0, layer_scores, agg_scores, layer_order,
                              agg_order, workspace, workspace_bytes, stream);
}

extern "C" int ct_score_chunks_band(const void* keys, const void* values, int dtype, int64_t C,
                                    int64_t L, int64_t N, int64_t lanes, int64_t ld_token,
                                    int64_t ld_layer, int64_t ld_chunk, int64_t cutoff,
                                    int precision, int band, double* layer_scores,
                                    double* agg_scores, int32_t* layer_order,
                                    int32_t* agg_order, void* workspace, size_t workspace_bytes,
                                    void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (band != 0 && band != 1) return fail(CT_ERR_PARAM, "band %d", band);
  if (C < 1 || L < 1 || N < 1 || lanes < 1)
    return fail(CT_ERR_SHAPE, "score geometry C=%lld L=%lld N=%lld lanes=%lld", (long long)C,
                (long long)L, (long long)N, (long long)lanes);
  if (!valid_dtype(dtype)) return fail(CT_ERR_PARAM, "dtype %d", dtype);
  if (precision != CT_F64 && precision != CT_F32) return fail(CT_ERR_PARAM, "precision %d", precision);
  if (cutoff < 0 || cutoff > N / 2 + 1) return fail(CT_ERR_PARAM, "cutoff %lld", (long long)cutoff);
  if (!keys || !values || !layer_scores) return fail(CT_ERR_PARAM, "null tensor");
  if (C * L > 65535) return fail(CT_ERR_UNSUPPORTED, "C*L too large");
  const int cut = band ? -(int)(cutoff + 1) : (int)cutoff;  // kernels: <0 = high band
  if (workspace_bytes < ct_score_workspace_bytes(C, L, N, lanes, precision))
    return fail(CT_ERR_PARAM, "workspace too small");
  const int nlb = (int)((lanes + LANE_BLOCK - 1) / LANE_BLOCK);
  char* ws = (char*)workspace;
  double* partial = (double*)ws;
  ws += align_up((size_t)C * L * 2 * nlb * N * sizeof(double), 256);
  void* tw_d = ws;
  ws += align_up((size_t)N * sizeof(cpx<double>), 256);
  void* tw_f = ws;
  int rc;
  if (fft_path(N)) {
    const int lg = ilog2_exact(N);
    twiddle_table<<<(unsigned)((N + 255) / 256), 256, 0, st>>>((int)N, (cpx<double>*)tw_d,
                                                                (cpx<float>*)tw_f);
    if ((rc = check_launch("twiddle_table"))) return rc;
    if (precision == CT_F64) {
      rc = dtype == CT_F32
               ? launch_fft<double, float>(lg, keys, values, (int)L, (int)C, (int)lanes, ld_token,
                                           ld_layer, ld_chunk, cut, tw_d, partial, st)
               : launch_fft<double, __nv_bfloat16>(lg, keys, values, (int)L, (int)C, (int)lanes,
                                                   ld_token, ld_layer, ld_chunk, cut, tw_d,
                                                   partial, st);
    } else {
      rc = dtype == CT_F32
               ? launch_fft<float, float>(lg, keys, values, (int)L, (int)C, (int)lanes, ld_token,
                                          ld_layer, ld_chunk, cut, tw_f, partial, st)
               : launch_fft<float, __nv_bfloat16>(lg, keys, values, (int)L, (int)C, (int)lanes,
                                                  ld_token, ld_layer, ld_chunk, cut, tw_f,
                                                  partial, st);
    }
    if (rc) return rc;
  } else if (MrPlan plan; mr_plan(N, &plan)) {
    twiddle_table<<<(unsigned)((N + 255) / 256), 256, 0, st>>>((int)N, (cpx<double>*)tw_d,
                                                                (cpx<float>*)tw_f);
    if ((rc = check_launch("twiddle_table"))) return rc;
    if (precision == CT_F64)
      rc = dtype == CT_F32
               ? launch_mr<double, float>(keys, values, N, (int)L, (int)C, (int)lanes, ld_token,
                                          ld_layer, ld_chunk, cut, tw_d, plan, partial, st)
               : launch_mr<double, __nv_bfloat16>(keys, values, N, (int)L, (int)C, (int)lanes,
                                                  ld_token, ld_layer, ld_chunk, cut, tw_d, plan,
                                                  partial, st);
    else
      rc = dtype == CT_F32
               ? launch_mr<float, float>(keys, values, N, (int)L, (int)C, (int)lanes, ld_token,
                                         ld_layer, ld_chunk, cut, tw_f, plan, partial, st)
               : launch_mr<float, __nv_bfloat16>(keys, values, N, (int)L, (int)C, (int)lanes,
                                                 ld_token, ld_layer, ld_chunk, cut, tw_f, plan,
                                                 partial, st);
    if (rc) return rc;
  } else {
    double* p = (double*)tw_d;
    lowpass_kernel_table<<<(unsigned)((N + 255) / 256), 256, 0, st>>>((int)N, cut, p);
    if ((rc = check_launch("lowpass_kernel_table"))) return rc;
    dim3 grid((unsigned)((N + 31) / 32), (unsigned)(2 * nlb), (unsigned)(C * L));
    if (dtype == CT_F32)
      direct_energy_kernel<float><<<grid, 256, 0, st>>>((const float*)keys, (const float*)values,
                                                        (int)N, (int)L, (int)lanes, ld_token,
                                                        ld_layer, ld_chunk, p, nlb, partial);
    else
      direct_energy_kernel<__nv_bfloat16><<<grid, 256, 0, st>>>(
          (const __nv_bfloat16*)keys, (const __nv_bfloat16*)values, (int)N, (int)L, (int)lanes,
          ld_token, ld_layer, ld_chunk, p, nlb, partial);
    if ((rc = check_launch("direct_energy_kernel"))) return rc;
  }
  const int64_t total = C * N;
  combine_scores<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(partial, (int)C, (int)L, (int)N,
                                                                  nlb, layer_scores, agg_scores);
  if ((rc = check_launch("combine_scores"))) return rc;
  if (layer_order && (rc = ct_desc_order(layer_scores, C * L, N, layer_order, stream))) return rc;
  if (agg_order) {
    if (!agg_scores) return fail(CT_ERR_PARAM, "agg_order needs agg_scores");
    if ((rc = ct_desc_order(agg_scores, C, N, agg_order, stream))) return rc;
  }
  return CT_OK;
}

extern "C" int ct_selection_plan(const int32_t* agg_orders, const int64_t* offsets,
                                 const int64_t* ks, const int64_t* rec_base,
                                 const int64_t* keep_base, int64_t n_chunks,
                                 int64_t max_chunk_tokens, int32_t* rec_global,
                                 int32_t* keep_global, int32_t* keep_src_row, void* stream) {
  if (n_chunks < 1) return fail(CT_ERR_PLAN, "need at least one chunk");
  const size_t smem = (size_t)max_chunk_tokens * sizeof(int);
  if (smem > 200 * 1024) return fail(CT_ERR_UNSUPPORTED, "chunk of %lld tokens", (long long)max_chunk_tokens);
  CT_CUDA(cudaFuncSetAttribute(selection_plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  selection_plan_kernel<<<(unsigned)n_chunks, PLAN_THREADS, smem, (cudaStream_t)stream>>>(
      agg_orders, offsets, ks, rec_base, keep_base, rec_global, keep_global, keep_src_row);
  return check_launch("selection_plan_kernel");
}

// ct/spectral.py:162-184 for one chunk: k = min(max(ceil(r N - 1e-9), 0), N)
// (the reference's float guard, same double arithmetic); the first k entries
// of `order` ascending -> sel [k], the rest ascending -> keep [N - k].
extern "C" int ct_select(const int32_t* order, int64_t n, double r, int32_t* sel, int32_t* keep,
                         int64_t* k_out, void* stream) {
  if (!(r >= 0.0 && r <= 1.0)) return fail(CT_ERR_PARAM, "ratio must be in [0, 1], got %g", r);
  if (n < 0) return fail(CT_ERR_SHAPE, "negative token count %lld", (long long)n);
  int64_t k = (int64_t)ceil(r * (double)n - 1e-9);
  k = k < 0 ? 0 : (k > n ? n : k);
  if (k_out) *k_out = k;
  if (n == 0) return CT_OK;
  const size_t smem = (size_t)n * sizeof(int);
  if (smem > 200 * 1024) return fail(CT_ERR_UNSUPPORTED, "chunk of %lld tokens", (long long)n);
  CT_CUDA(cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
  select_kernel<<<1, PLAN_THREADS, smem, (cudaStream_t)stream>>>(order, (int)n, (int)k, sel, keep);
  return check_launch("select_kernel");
}

// One chunk of L layers [L][N][ld_token] (lanes = H*D), exact (f64) mode, with
// the reference's cutoff floor(alpha * (N/2 + 1)) (ct/spectral.py:57-58,82-90).
extern "C" int ct_score_chunk(const void* keys, const void* values, int dtype, int64_t L,
                              int64_t N, int64_t H, int64_t D, int64_t ld_token, double alpha,
                              double* layer_scores, double* agg_scores, int32_t* agg_order,
                              void* workspace, size_t workspace_bytes, void* stream) {
  if (!(alpha >= 0.0 && alpha <= 1.0))
    return fail(CT_ERR_PARAM, "alpha must be in [0, 1], got %g", alpha);
  if (H < 1 || D < 1) return fail(CT_ERR_SHAPE, "H=%lld D=%lld", (long long)H, (long long)D);
  const int64_t cutoff = (int64_t)floor(alpha * (double)(N / 2 + 1));
  return ct_score_chunks(keys, values, dtype, 1, L, N, H * D, ld_token, N * ld_token,
                         L * N * ld_token, cutoff, CT_F64, layer_scores, agg_scores, nullptr,
                         agg_order, workspace, workspace_bytes, stream);
}
