// (2)+(3) sparse gather + deferred RoPE + blend, and (4) QKV rope/scatter
// epilogue.  Replaces ct/rope.py:42-81 (RopeParams.freqs / rope_rotate /
// rope_apply), the reuse half of ct/pipesim.py:322-357 (fuse_layer), the
// in-path gather of ct/toymodel.py:269-283 and the recompute half of
// ct/toymodel.py:157-172.
//
// All kernels are HBM-bound row movers: one "unit" = VEC rotation pairs of
// one head of one row (8 bf16 = 16 B per K/V access for adjacent pairing),
// rows are walked grid-stride, and (cos, sin) comes from an L2-resident
// [pos][D/2] table built once in float64 (F7: fp32 angles break at 64K).
// fp32 mode (f32 caches) rotates in float64 with the unfused product/sum of
// ct/rope.py:61-62 and rounds once to f32, reproducing the reference bits.
#include "common.cuh"

namespace ct {

__global__ void rope_table_kernel(const double* __restrict__ freqs, int half, int64_t n_pos,
                                  double scaling, const int64_t* __restrict__ positions,
                                  double2* __restrict__ td, float2* __restrict__ tf) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n_pos * half) return;
  const int64_t p = positions ? positions[t / half] : t / half;
  const int j = (int)(t % half);
  // angles = outer(positions.astype(f64) * scaling, freqs)  (ct/rope.py:53-54)
  const double ang = __dmul_rn(__dmul_rn((double)p, scaling), freqs[j]);
  double s, c;
  sincos(ang, &s, &c);
  if (td) td[t] = make_double2(c, s);
  if (tf) tf[t] = make_float2((float)c, (float)s);
}

// Rotate one group of VEC pairs.  a[i], b[i] are the pair members.
template <int VEC>
__device__ __forceinline__ void rotate_f64(float* a, float* b, const double2* cs) {
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const double x = a[i], y = b[i];
    const double c = cs[i].x, s = cs[i].y;
    const double ra = __dsub_rn(__dmul_rn(x, c), __dmul_rn(y, s));
    const double rb = __dadd_rn(__dmul_rn(x, s), __dmul_rn(y, c));
    a[i] = (float)ra;
    b[i] = (float)rb;
  }
}
template <int VEC>
__device__ __forceinline__ void rotate_f32(float* a, float* b, const float2* cs) {
#pragma unroll
  for (int i = 0; i < VEC; ++i) {
    const float x = a[i], y = b[i];
    a[i] = x * cs[i].x - y * cs[i].y;
    b[i] = x * cs[i].y + y * cs[i].x;
  }
}

// Element offsets of pair group (head h, first pair j0) inside a row.
// adjacent: elements 2j, 2j+1; split: j, j + D/2.
template <typename T, int VEC>
__device__ __forceinline__ void load_pairs(const T* row, int h, int j0, int D, int pairing,
                                           float* a, float* b) {
  const T* hp = row + (int64_t)h * D;
  if (pairing == CT_ROPE_ADJACENT) {
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      a[i] = to_f32(hp[2 * (j0 + i)]);
      b[i] = to_f32(hp[2 * (j0 + i) + 1]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      a[i] = to_f32(hp[j0 + i]);
      b[i] = to_f32(hp[j0 + i + D / 2]);
    }
  }
}
template <typename T, int VEC>
__device__ __forceinline__ void store_pairs(T* row, int h, int j0, int D, int pairing,
                                            const float* a, const float* b) {
  T* hp = row + (int64_t)h * D;
  if (pairing == CT_ROPE_ADJACENT) {
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      hp[2 * (j0 + i)] = from_f32<T>(a[i]);
      hp[2 * (j0 + i) + 1] = from_f32<T>(b[i]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < VEC; ++i) {
      hp[j0 + i] = from_f32<T>(a[i]);
      hp[j0 + i + D / 2] = from_f32<T>(b[i]);
    }
  }
}

// 16-byte vectorised specialisation for bf16 adjacent pairs (VEC = 4).
__device__ __forceinline__ void load8_bf16(const __nv_bfloat16* p, float* a, float* b) {
  const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
  const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h2[i]);
    a[i] = f.x;
    b[i] = f.y;
  }
}
__device__ __forceinline__ void store8_bf16(__nv_bfloat16* p, const float* a, const float* b) {
  uint4 u;
  __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h2[i] = __floats2bfloat162_rn(a[i], b[i]);
  *reinterpret_cast<uint4*>(p) = u;
}

template <typename T, int VEC>
__device__ __forceinline__ void rot_unit(const T* src, T* dst, int h, int j0, int D,
                                         int pairing, const void* table, int64_t pos,
                                         bool f64math) {
  float a[VEC], b[VEC];
  const int half = D / 2;
  if constexpr (sizeof(T) == 2 && VEC == 4) {
    if (pairing == CT_ROPE_ADJACENT) {
      load8_bf16(reinterpret_cast<const __nv_bfloat16*>(src) + (int64_t)h * D + 2 * j0, a, b);
    } else {
      load_pairs<T, VEC>(src, h, j0, D, pairing, a, b);
    }
  } else {
    load_pairs<T, VEC>(src, h, j0, D, pairing, a, b);
  }
  if (f64math) {
    const double2* cs = reinterpret_cast<const double2*>(table) + pos * half + j0;
    double2 c[VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i) c[i] = __ldg(cs + i);
    rotate_f64<VEC>(a, b, c);
  } else {
    const float2* cs = reinterpret_cast<const float2*>(table) + pos * half + j0;
    float2 c[VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i) c[i] = __ldg(cs + i);
    rotate_f32<VEC>(a, b, c);
  }
  if constexpr (sizeof(T) == 2 && VEC == 4) {
    if (pairing == CT_ROPE_ADJACENT) {
      store8_bf16(reinterpret_cast<__nv_bfloat16*>(dst) + (int64_t)h * D + 2 * j0, a, b);
      return;
    }
  }
  store_pairs<T, VEC>(dst, h, j0, D, pairing, a, b);
}

template <typename T, int VEC>
__device__ __forceinline__ void copy_unit(const T* src, T* dst, int h, int j0, int D,
                                          int pairing) {
  if constexpr (sizeof(T) == 2 && VEC == 4) {
    if (pairing == CT_ROPE_ADJACENT) {
      const int64_t o = (int64_t)h * D + 2 * j0;
      *reinterpret_cast<uint4*>(dst + o) = __ldg(reinterpret_cast<const uint4*>(src + o));
      return;
    }
  }
  float a[VEC], b[VEC];
  load_pairs<T, VEC>(src, h, j0, D, pairing, a, b);
  store_pairs<T, VEC>(dst, h, j0, D, pairing, a, b);
}

struct SegArray {
  ct_segment s[CT_MAX_SEGMENTS];
};

// Rotate the 4 adjacent pairs packed in a 16-B bf16 chunk with (cos, sin)[4].
__device__ __forceinline__ uint4 rot8_bf16(uint4 u, const float4 c01, const float4 c23) {
  __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
  const float cs[8] = {c01.x, c01.y, c01.z, c01.w, c23.x, c23.y, c23.z, c23.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 f = __bfloat1622float2(h2[i]);
    const float c = cs[2 * i], s = cs[2 * i + 1];
    h2[i] = __floats2bfloat162_rn(f.x * c - f.y * s, f.x * s + f.y * c);
  }
  return u;
}

// Hot-path blend for bf16 caches with adjacent pairing.  One thread owns one
// 16-B column chunk c (4 rotation pairs) of one reused row and walks the row's
// heads: the (cos, sin) of (pos, pairs 4c..4c+3) is loaded ONCE and shared by
// all H heads (the table is per position, not per head), and all 2*HB K/V
// loads of a head block are issued before any math, so 2*HB*16 B are in
// flight per thread.  A warp covers 2 rows x 16 chunks: every load/store
// instruction moves two contiguous 256-B row segments.
template <int HB>
__global__ void __launch_bounds__(256)
blend_bf16_kernel(SegArray segs, int64_t src_row_stride, int H, int cph,
                  const float4* __restrict__ table, int half, __nv_bfloat16* __restrict__ kc,
                  __nv_bfloat16* __restrict__ vc, int64_t cache_row_stride) {
  const ct_segment sg = segs.s[blockIdx.y];
  const int64_t total = sg.rows * cph;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const __nv_bfloat16* ks = reinterpret_cast<const __nv_bfloat16*>(sg.k);
  const __nv_bfloat16* vs = reinterpret_cast<const __nv_bfloat16*>(sg.v);
  const int D = 8 * cph;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total; u += nthr) {
    const int64_t row = u / cph;
    const int c = (int)(u - row * cph);
    const int32_t tk = __ldg(sg.tok + row);
    const int64_t pos = sg.pos0 + tk;
    const int64_t srow = sg.src_by_tok ? (int64_t)tk : row;
    const float4* t = table + (pos * half + 4 * c) / 2;
    const float4 c0 = __ldg(t), c1 = __ldg(t + 1);
    const uint4* kin = reinterpret_cast<const uint4*>(ks + srow * src_row_stride + 8 * c);
    const uint4* vin = reinterpret_cast<const uint4*>(vs + srow * src_row_stride + 8 * c);
    uint4* kout = reinterpret_cast<uint4*>(kc + pos * cache_row_stride + 8 * c);
    uint4* vout = reinterpret_cast<uint4*>(vc + pos * cache_row_stride + 8 * c);
    const int hstride = D / 8;  // uint4 per head
    for (int h0 = 0; h0 < H; h0 += HB) {
      uint4 kr[HB], vr[HB];
#pragma unroll
      for (int h = 0; h < HB; ++h) {
        if (h0 + h < H) {
          kr[h] = ldg_stream(kin + (h0 + h) * hstride);
          vr[h] = ldg_stream(vin + (h0 + h) * hstride);
        }
      }
#pragma unroll
      for (int h = 0; h < HB; ++h) {
        if (h0 + h < H) {
          kout[(h0 + h) * hstride] = rot8_bf16(kr[h], c0, c1);
          vout[(h0 + h) * hstride] = vr[h];
        }
      }
    }
  }
}

// Hot-path QKV epilogue for bf16 in/out, adjacent pairing.  One thread owns
// 16-B column chunk c of a block of HB consecutive heads of one qkv row; the
// (cos, sin) of (pos, pairs 4c..4c+3) is loaded once per thread and shared by
// the block's q/k heads.  q heads -> q_out (rotated), k -> cache (rotated) +
// optional raw copy, v -> cache.
template <int HB>
__global__ void __launch_bounds__(256)
qkv_bf16_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t ld_qkv,
                const int32_t* __restrict__ positions, int64_t A, int Hq, int Hkv, int D,
                const float4* __restrict__ table, __nv_bfloat16* __restrict__ q_out,
                __nv_bfloat16* __restrict__ kc, __nv_bfloat16* __restrict__ vc,
                int64_t crs, __nv_bfloat16* __restrict__ k_raw) {
  const int cph = D / 8;
  const int hpr = Hq + 2 * Hkv;
  const int ng = (hpr + HB - 1) / HB;
  const int half = D / 2;
  const int64_t total = A * ng * cph;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total; u += nthr) {
    const int64_t ag = u / cph;
    const int c = (int)(u - ag * cph);
    const int64_t a = ag / ng;
    const int h0 = (int)(ag - a * ng) * HB;
    const int64_t pos = __ldg(positions + a);
    const uint4* in = reinterpret_cast<const uint4*>(qkv + a * ld_qkv + 8 * c);
    float4 c0 = make_float4(0.f, 0.f, 0.f, 0.f), c1 = c0;
    if (h0 < Hq + Hkv) {
      const float4* t = table + (pos * half + 4 * c) / 2;
      c0 = __ldg(t);
      c1 = __ldg(t + 1);
    }
    uint4 x[HB];
#pragma unroll
    for (int h = 0; h < HB; ++h)
      if (h0 + h < hpr) x[h] = ldg_stream(in + (h0 + h) * cph);
#pragma unroll
    for (int h = 0; h < HB; ++h) {
      const int hh = h0 + h;
      if (hh >= hpr) break;
      if (hh >= Hq + Hkv) {
        *reinterpret_cast<uint4*>(vc + pos * crs + (int64_t)(hh - Hq - Hkv) * D + c * 8) = x[h];
        continue;
      }
      const uint4 r = rot8_bf16(x[h], c0, c1);
      if (hh < Hq) {
        *reinterpret_cast<uint4*>(q_out + (a * Hq + hh) * (int64_t)D + c * 8) = r;
      } else {
        *reinterpret_cast<uint4*>(kc + pos * crs + (int64_t)(hh - Hq) * D + c * 8) = r;
        if (k_raw)
          *reinterpret_cast<uint4*>(k_raw + (a * Hkv + hh - Hq) * (int64_t)D + c * 8) = x[h];
      }
    }
  }
}

// grid: x = row blocks, y = segment.  256 threads; units per row = H*(D/2)/VEC.
template <typename T, int VEC>
__global__ void __launch_bounds__(256)
gather_rope_blend_kernel(SegArray segs, int64_t src_row_stride, int H, int D, int pairing,
                         const void* __restrict__ table, T* __restrict__ kc,
                         T* __restrict__ vc, int64_t cache_row_stride, bool f64math) {
  const ct_segment sg = segs.s[blockIdx.y];
  const int upr = H * (D / 2) / VEC;  // units per row
  const int64_t total = sg.rows * upr;
  const T* ks = reinterpret_cast<const T*>(sg.k);
  const T* vs = reinterpret_cast<const T*>(sg.v);
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = u / upr;
    const int w = (int)(u % upr);
    const int h = w / ((D / 2) / VEC);
    const int j0 = (w % ((D / 2) / VEC)) * VEC;
    const int32_t tk = __ldg(sg.tok + row);
    const int64_t pos = sg.pos0 + tk;
    const int64_t srow = sg.src_by_tok ? (int64_t)tk : row;
    const T* ksrc = ks + srow * src_row_stride;
    const T* vsrc = vs + srow * src_row_stride;
    rot_unit<T, VEC>(ksrc, kc + pos * cache_row_stride, h, j0, D, pairing, table, pos, f64math);
    copy_unit<T, VEC>(vsrc, vc + pos * cache_row_stride, h, j0, D, pairing);
  }
}

template <typename T, int VEC>
__global__ void __launch_bounds__(256)
rope_apply_kernel(const T* __restrict__ x, const int32_t* __restrict__ positions, int64_t n,
                  int H, int D, int pairing, const void* __restrict__ table, T* __restrict__ out,
                  bool f64math) {
  const int upr = H * (D / 2) / VEC;
  const int64_t total = n * upr;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = u / upr;
    const int w = (int)(u % upr);
    const int h = w / ((D / 2) / VEC);
    const int j0 = (w % ((D / 2) / VEC)) * VEC;
    const int64_t pos = positions[row];
    const int64_t ro = row * (int64_t)H * D;
    rot_unit<T, VEC>(x + ro, out + ro, h, j0, D, pairing, table, pos, f64math);
  }
}

// QKV epilogue.  Heads [0,Hq) -> q_out (rotated), [Hq, Hq+Hkv) -> k (rotated
// into k_cache[pos], raw into k_raw_out[a]), [Hq+Hkv, Hq+2Hkv) -> v_cache[pos].
template <typename TI, typename TQ, typename TC, int VEC>
__global__ void __launch_bounds__(256)
qkv_rope_scatter_kernel(const TI* __restrict__ qkv, int64_t ld_qkv,
                        const int32_t* __restrict__ positions, int64_t A, int Hq, int Hkv, int D,
                        int pairing, const void* __restrict__ table, TQ* __restrict__ q_out,
                        TC* __restrict__ kc, TC* __restrict__ vc, int64_t cache_row_stride,
                        TC* __restrict__ k_raw_out, bool f64math) {
  const int hpr = Hq + 2 * Hkv;
  const int gph = (D / 2) / VEC;
  const int upr = hpr * gph;
  const int64_t total = A * upr;
  const int half = D / 2;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = u / upr;
    const int w = (int)(u % upr);
    const int hh = w / gph;
    const int j0 = (w % gph) * VEC;
    const int64_t pos = positions[a];
    const TI* row = qkv + a * ld_qkv;
    float x[VEC], y[VEC];
    load_pairs<TI, VEC>(row, hh, j0, D, pairing, x, y);
    if (hh >= Hq + Hkv) {  // value: copy
      store_pairs<TC, VEC>(vc + pos * cache_row_stride, hh - Hq - Hkv, j0, D, pairing, x, y);
      continue;
    }
    if (hh >= Hq && k_raw_out)
      store_pairs<TC, VEC>(k_raw_out + a * (int64_t)Hkv * D, hh - Hq, j0, D, pairing, x, y);
    if (f64math) {
      const double2* cs = reinterpret_cast<const double2*>(table) + pos * half + j0;
      double2 c[VEC];
#pragma unroll
      for (int i = 0; i < VEC; ++i) c[i] = cs[i];
      rotate_f64<VEC>(x, y, c);
    } else {
      const float2* cs = reinterpret_cast<const float2*>(table) + pos * half + j0;
      float2 c[VEC];
#pragma unroll
      for (int i = 0; i < VEC; ++i) c[i] = cs[i];
      rotate_f32<VEC>(x, y, c);
    }
    if (hh < Hq)
      store_pairs<TQ, VEC>(q_out + a * (int64_t)Hq * D, hh, j0, D, pairing, x, y);
    else
      store_pairs<TC, VEC>(kc + pos * cache_row_stride, hh - Hq, j0, D, pairing, x, y);
  }
}

__global__ void rows_copy_kernel(const uint32_t* __restrict__ src, const int32_t* __restrict__ idx,
                                 int64_t n, int64_t words, uint32_t* __restrict__ dst,
                                 bool scatter) {
  const int64_t total = n * words;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / words, w = t % words;
    const int64_t j = idx[i];
    if (scatter)
      dst[j * words + w] = src[i * words + w];
    else
      dst[i * words + w] = src[j * words + w];
  }
}


// Importance-ordered pool image (offline stage): one warp per destination
// (chunk, layer, rank p) moves the K row then the V row of token order[c][p].
// W = uint4 (16-byte rows) or uint32_t; VPL > 0: the row is VPL vectors per
// lane and all 2*VPL loads are issued before the streaming stores (16 KiB in
// flight per warp-row at VPL = 4), VPL = 0: generic lane loop.  Every byte
// crosses HBM once in each direction.  dst[((c L + l) N + p) 2 + side][row].
template <typename W>
__device__ __forceinline__ W ld_once(const W* p) { return __ldg(p); }
template <>
__device__ __forceinline__ uint4 ld_once<uint4>(const uint4* p) { return ldg_stream(p); }

template <typename W, int VPL>
__global__ void __launch_bounds__(256)
pool_permute_kernel(const W* __restrict__ keys, const W* __restrict__ values, int C, int L, int N,
                    int64_t ld_token, int64_t ld_layer, int64_t ld_chunk, int vec,
                    const int32_t* __restrict__ order, W* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t total = (int64_t)C * L * N;
  for (int64_t u = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); u < total;
       u += warps) {
    const int p = (int)(u % N);
    const int64_t cl = u / N;
    const int l = (int)(cl % L), c = (int)(cl / L);
    const int64_t src =
        c * ld_chunk + l * ld_layer + (int64_t)__ldg(order + (int64_t)c * N + p) * ld_token;
    W* out = dst + u * 2 * vec;
    if constexpr (VPL > 0) {
      W k[VPL], v[VPL];
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        k[i] = ld_once(keys + src + lane + 32 * i);
        v[i] = ld_once(values + src + lane + 32 * i);
      }
#pragma unroll
      for (int i = 0; i < VPL; ++i) {
        __stcs(out + lane + 32 * i, k[i]);
        __stcs(out + vec + lane + 32 * i, v[i]);
      }
    } else {
      for (int w = lane; w < vec; w += 32) {
        const W k = ld_once(keys + src + w), v = ld_once(values + src + w);
        __stcs(out + w, k);
        __stcs(out + vec + w, v);
      }
    }
  }
}

static unsigned grid_for(int64_t units, int threads) {
  int64_t b = (units + threads - 1) / threads;
  const int64_t cap = 148 * 32;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (unsigned)b;
}

}  // namespace ct

using namespace ct;

extern "C" int ct_rope_table(const double* freqs, int64_t half_dim, int64_t n_pos,
                             double scaling, const int64_t* positions, void* table_f64,
                             void* table_f32, void* stream) {
  if (half_dim < 1 || n_pos < 0) return fail(CT_ERR_SHAPE, "rope table geometry");
  if (n_pos == 0) return CT_OK;
  const int64_t total = half_dim * n_pos;
  rope_table_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      freqs, (int)half_dim, n_pos, scaling, positions, (double2*)table_f64, (float2*)table_f32);
  return check_launch("rope_table_kernel");
}

// f64 rows in and out (ct/rope.py:47-72 rope_rotate, which returns float64):
// ra = a cos - b sin, rb = a sin + b cos as separate correctly rounded
// products and sums (no FMA contraction), like numpy's elementwise ops.
__global__ void __launch_bounds__(256)
rope_rotate_f64_kernel(const double* __restrict__ x, const int32_t* __restrict__ positions,
                       int64_t n, int H, int D, int pairing, const double2* __restrict__ table,
                       double* __restrict__ out) {
  const int half = D / 2;
  const int64_t total = n * H * half;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < total;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = u / (H * half);
    const int rem = (int)(u % (H * half));
    const int h = rem / half, j = rem % half;
    const double2 cs = __ldg(table + (int64_t)positions[row] * half + j);
    const int ia = pairing == CT_ROPE_ADJACENT ? 2 * j : j;
    const int ib = pairing == CT_ROPE_ADJACENT ? 2 * j + 1 : j + half;
    const int64_t base = (row * H + h) * (int64_t)D;
    const double a = x[base + ia], b = x[base + ib];
    out[base + ia] = __dsub_rn(__dmul_rn(a, cs.x), __dmul_rn(b, cs.y));
    out[base + ib] = __dadd_rn(__dmul_rn(a, cs.y), __dmul_rn(b, cs.x));
  }
}

extern "C" int ct_rope_apply(const void* x, const int32_t* positions, int64_t n, int64_t H,
                             int64_t D, int dtype, int pairing, const void* table, void* out,
                             void* stream) {
  if (D < 2 || D % 2) return fail(CT_ERR_SHAPE, "head_dim must be even, got %lld", (long long)D);
  if (!valid_dtype(dtype) && dtype != CT_F64) return fail(CT_ERR_PARAM, "dtype %d", dtype);
  if (pairing != CT_ROPE_ADJACENT && pairing != CT_ROPE_SPLIT) return fail(CT_ERR_PARAM, "pairing");
  if (n == 0) return CT_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == CT_F64) {
    rope_rotate_f64_kernel<<<grid_for(n * H * (D / 2), 256), 256, 0, st>>>(
        (const double*)x, positions, n, (int)H, (int)D, pairing, (const double2*)table,
        (double*)out);
    return check_launch("rope_rotate_f64_kernel");
  }
  const bool f64m = dtype == CT_F32;
  const bool v4 = (D / 2) % 4 == 0;
  const int64_t units = n * H * (D / 2) / (v4 ? 4 : 1);
  const unsigned g = grid_for(units, 256);
  if (dtype == CT_F32) {
    if (v4) rope_apply_kernel<float, 4><<<g, 256, 0, st>>>((const float*)x, positions, n, (int)H, (int)D, pairing, table, (float*)out, f64m);
    else rope_apply_kernel<float, 1><<<g, 256, 0, st>>>((const float*)x, positions, n, (int)H, (int)D, pairing, table, (float*)out, f64m);
  } else {
    if (v4) rope_apply_kernel<__nv_bfloat16, 4><<<g, 256, 0, st>>>((const __nv_bfloat16*)x, positions, n, (int)H, (int)D, pairing, table, (__nv_bfloat16*)out, f64m);
    else rope_apply_kernel<__nv_bfloat16, 1><<<g, 256, 0, st>>>((const __nv_bfloat16*)x, positions, n, (int)H, (int)D, pairing, table, (__nv_bfloat16*)out, f64m);
  }
  return check_launch("rope_apply_kernel");
}

extern "C" int ct_gather_rope_blend(const ct_segment* segs, int n_segs, int64_t src_row_stride,
                                    int64_t H, int64_t D, int dtype, int pairing,
                                    const void* table, void* k_cache, void* v_cache,
                                    int64_t cache_row_stride, void* stream) {
  if (n_segs < 0 || n_segs > CT_MAX_SEGMENTS) return fail(CT_ERR_PARAM, "n_segs %d", n_segs);
  if (D < 2 || D % 2) return fail(CT_ERR_SHAPE, "head_dim must be even");
  if (!valid_dtype(dtype)) return fail(CT_ERR_PARAM, "dtype %d", dtype);
  if (n_segs == 0) return CT_OK;
  SegArray arr;
  memset(&arr, 0, sizeof(arr));
  int64_t max_rows = 0;
  for (int i = 0; i < n_segs; ++i) {
    arr.s[i] = segs[i];
    if (segs[i].rows > max_rows) max_rows = segs[i].rows;
  }
  if (max_rows == 0) return CT_OK;
  cudaStream_t st = (cudaStream_t)stream;
  bool fast = dtype == CT_BF16 && pairing == CT_ROPE_ADJACENT && D % 8 == 0 &&
              src_row_stride % 8 == 0 && cache_row_stride % 8 == 0 &&
              ((uintptr_t)k_cache % 16 == 0) && ((uintptr_t)v_cache % 16 == 0) &&
              ((uintptr_t)table % 16 == 0);
  for (int i = 0; i < n_segs && fast; ++i)
    fast = ((uintptr_t)segs[i].k % 16 == 0) && ((uintptr_t)segs[i].v % 16 == 0);
  if (fast) {
    const int cph = (int)(D / 8);
    int64_t bx = (max_rows * cph + 255) / 256;
    const int64_t cap = (148 * 16 + n_segs - 1) / n_segs;
    if (bx > cap) bx = cap;
    dim3 grid((unsigned)bx, (unsigned)n_segs);
    blend_bf16_kernel<8><<<grid, 256, 0, st>>>(arr, src_row_stride, (int)H, cph,
                                               (const float4*)table, (int)(D / 2),
                                               (__nv_bfloat16*)k_cache, (__nv_bfloat16*)v_cache,
                                               cache_row_stride);
    return check_launch("blend_bf16_kernel");
  }
  const bool v4 = (D / 2) % 4 == 0;
  const int64_t upr = H * (D / 2) / (v4 ? 4 : 1);
  int64_t bx = (max_rows * upr + 255) / 256;
  const int64_t cap = (148 * 16 + n_segs - 1) / n_segs;
  if (bx > cap) bx = cap;
  dim3 grid((unsigned)bx, (unsigned)n_segs);
  const bool f64m = dtype == CT_F32;
  if (dtype == CT_F32) {
    if (v4) gather_rope_blend_kernel<float, 4><<<grid, 256, 0, st>>>(arr, src_row_stride, (int)H, (int)D, pairing, table, (float*)k_cache, (float*)v_cache, cache_row_stride, f64m);
    else gather_rope_blend_kernel<float, 1><<<grid, 256, 0, st>>>(arr, src_row_stride, (int)H, (int)D, pairing, table, (float*)k_cache, (float*)v_cache, cache_row_stride, f64m);
  } else {
    if (v4) gather_rope_blend_kernel<__nv_bfloat16, 4><<<grid, 256, 0, st>>>(arr, src_row_stride, (int)H, (int)D, pairing, table, (__nv_bfloat16*)k_cache, (__nv_bfloat16*)v_cache, cache_row_stride, f64m);
    else gather_rope_blend_kernel<__nv_bfloat16, 1><<<grid, 256, 0, st>>>(arr, src_row_stride, (int)H, (int)D, pairing, table, (__nv_bfloat16*)k_cache, (__nv_bfloat16*)v_cache, cache_row_stride, f64m);
  }
  return check_launch("gather_rope_blend_kernel");
}

template <typename TI, typename TQ, typename TC, int VEC>
static void launch_qkv(unsigned g, cudaStream_t st, const void* qkv, int64_t ld, const int32_t* pos,
                       int64_t A, int Hq, int Hkv, int D, int pairing, const void* table,
                       void* q_out, void* kc, void* vc, int64_t crs, void* kraw, bool f64m) {
  qkv_rope_scatter_kernel<TI, TQ, TC, VEC><<<g, 256, 0, st>>>(
      (const TI*)qkv, ld, pos, A, Hq, Hkv, D, pairing, table, (TQ*)q_out, (TC*)kc, (TC*)vc, crs,
      (TC*)kraw, f64m);
}

extern "C" int ct_qkv_rope_scatter(const void* qkv, int64_t ld_qkv, int in_dtype,
                                   const int32_t* positions, int64_t A, int64_t Hq, int64_t Hkv,
                                   int64_t D, int pairing, const void* table, void* q_out,
                                   int q_dtype, void* k_cache, void* v_cache, int cache_dtype,
                                   int64_t cache_row_stride, void* k_raw_out, void* stream) {
  if (D < 2 || D % 2) return fail(CT_ERR_SHAPE, "head_dim must be even");
  if (Hkv < 1 || Hq % Hkv) return fail(CT_ERR_SHAPE, "Hq=%lld not a multiple of Hkv=%lld", (long long)Hq, (long long)Hkv);
  if (!valid_dtype(in_dtype) || !valid_dtype(q_dtype) || !valid_dtype(cache_dtype))
    return fail(CT_ERR_PARAM, "dtype");
  if (A == 0) return CT_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (in_dtype == CT_BF16 && q_dtype == CT_BF16 && cache_dtype == CT_BF16 &&
      pairing == CT_ROPE_ADJACENT && D % 8 == 0 && ld_qkv % 8 == 0 &&
      cache_row_stride % 8 == 0 &&
      (((uintptr_t)qkv | (uintptr_t)q_out | (uintptr_t)k_cache | (uintptr_t)v_cache |
        (uintptr_t)table | (uintptr_t)k_raw_out) % 16 == 0)) {
    const int64_t units = A * ((Hq + 2 * Hkv + 7) / 8) * (D / 8);
    int64_t g = (units + 255) / 256;
    if (g > 148 * 16) g = 148 * 16;
    qkv_bf16_kernel<8><<<(unsigned)g, 256, 0, st>>>(
        (const __nv_bfloat16*)qkv, ld_qkv, positions, A, (int)Hq, (int)Hkv, (int)D,
        (const float4*)table, (__nv_bfloat16*)q_out, (__nv_bfloat16*)k_cache,
        (__nv_bfloat16*)v_cache, cache_row_stride, (__nv_bfloat16*)k_raw_out);
    return check_launch("qkv_bf16_kernel");
  }
  const bool v4 = (D / 2) % 4 == 0;
  const int64_t units = A * (Hq + 2 * Hkv) * (D / 2) / (v4 ? 4 : 1);
  const unsigned g = grid_for(units, 256);
  const bool f64m = cache_dtype == CT_F32;
  const int key = in_dtype * 100 + q_dtype * 10 + cache_dtype;
#define CT_QKV(TI, TQ, TC)                                                                       \
  if (v4) launch_qkv<TI, TQ, TC, 4>(g, st, qkv, ld_qkv, positions, A, (int)Hq, (int)Hkv, (int)D, \
                                    pairing, table, q_out, k_cache, v_cache, cache_row_stride,   \
                                    k_raw_out, f64m);                                            \
  else launch_qkv<TI, TQ, TC, 1>(g, st, qkv, ld_qkv, positions, A, (int)Hq, (int)Hkv, (int)D,    \
                                 pairing, table, q_out, k_cache, v_cache, cache_row_stride,      \
                                 k_raw_out, f64m);
  switch (key) {
    case CT_F32 * 100 + CT_F32 * 10 + CT_F32: CT_QKV(float, float, float) break;
    case CT_BF16 * 100 + CT_BF16 * 10 + CT_BF16: CT_QKV(__nv_bfloat16, __nv_bfloat16, __nv_bfloat16) break;
    case CT_F32 * 100 + CT_BF16 * 10 + CT_BF16: CT_QKV(float, __nv_bfloat16, __nv_bfloat16) break;
    case CT_BF16 * 100 + CT_F32 * 10 + CT_F32: CT_QKV(__nv_bfloat16, float, float) break;
    default: return fail(CT_ERR_UNSUPPORTED, "qkv dtype combination %d", key);
  }
#undef CT_QKV
  return check_launch("qkv_rope_scatter_kernel");
}

extern "C" int ct_scatter_rows(const void* src, const int32_t* idx, int64_t n, int64_t row_bytes,
                               void* dst, void* stream) {
  if (row_bytes % 4) return fail(CT_ERR_PARAM, "row_bytes %% 4");
  if (n == 0) return CT_OK;
  const int64_t words = row_bytes / 4;
  rows_copy_kernel<<<grid_for(n * words, 256), 256, 0, (cudaStream_t)stream>>>(
      (const uint32_t*)src, idx, n, words, (uint32_t*)dst, true);
  return check_launch("rows_copy_kernel");
}

extern "C" int ct_gather_rows(const void* src, const int32_t* idx, int64_t n, int64_t row_bytes,
                              void* dst, void* stream) {
  if (row_bytes % 4) return fail(CT_ERR_PARAM, "row_bytes %% 4");
  if (n == 0) return CT_OK;
  const int64_t words = row_bytes / 4;
  rows_copy_kernel<<<grid_for(n * words, 256), 256, 0, (cudaStream_t)stream>>>(
      (const uint32_t*)src, idx, n, words, (uint32_t*)dst, false);
  return check_launch("rows_copy_kernel");
}

extern "C" int ct_pool_permute(const void* keys, const void* values, int C, int L, int N,
                               int64_t ld_token, int64_t ld_layer, int64_t ld_chunk,
                               int64_t row_bytes, const int32_t* order, void* dst, void* stream) {
  if (C < 0 || L < 0 || N < 0) return fail(CT_ERR_SHAPE, "ct_pool_permute: negative geometry");
  if (row_bytes <= 0 || row_bytes % 4 || ld_token % 4 || ld_layer % 4 || ld_chunk % 4)
    return fail(CT_ERR_PARAM, "ct_pool_permute: row bytes and strides must be multiples of 4");
  if (ld_token < row_bytes) return fail(CT_ERR_SHAPE, "ct_pool_permute: token stride < row bytes");
  if (((uintptr_t)keys | (uintptr_t)values | (uintptr_t)dst) & 3)
    return fail(CT_ERR_PARAM, "ct_pool_permute: pointers must be 4-byte aligned");
  if ((int64_t)C * L * N == 0) return CT_OK;
  if (!keys || !values || !order || !dst) return fail(CT_ERR_PARAM, "ct_pool_permute: null pointer");
  const int64_t warps = (int64_t)C * L * N;
  int64_t blocks = (warps + 7) / 8;
  const int64_t cap = 148 * 8;
  if (blocks > cap) blocks = cap;
  cudaStream_t st = (cudaStream_t)stream;
  const bool v16 = row_bytes % 16 == 0 && ld_token % 16 == 0 && ld_layer % 16 == 0 &&
                   ld_chunk % 16 == 0 && !(((uintptr_t)keys | (uintptr_t)values | (uintptr_t)dst) & 15);
  if (v16) {
    const int vec = (int)(row_bytes / 16);
    auto args = [&](auto kern) {
      kern<<<(unsigned)blocks, 256, 0, st>>>((const uint4*)keys, (const uint4*)values, C, L, N,
                                             ld_token / 16, ld_layer / 16, ld_chunk / 16, vec,
                                             order, (uint4*)dst);
    };
    if (vec == 128)
      args(pool_permute_kernel<uint4, 4>);
    else if (vec == 256)
      args(pool_permute_kernel<uint4, 8>);
    else
      args(pool_permute_kernel<uint4, 0>);
  } else {
    pool_permute_kernel<uint32_t, 0><<<(unsigned)blocks, 256, 0, st>>>(
        (const uint32_t*)keys, (const uint32_t*)values, C, L, N, ld_token / 4, ld_layer / 4,
        ld_chunk / 4, (int)(row_bytes / 4), order, (uint32_t*)dst);
  }
  return check_launch("pool_permute_kernel");
}
