/*
 * cachetune_b200.h -- C ABI of the B200-native CacheTune online
 * selective-recompute prefill path (libcachetune_b200.so, sm_100a).
 *
 * Every entry point replaces one reference function on the hot path; the
 * reference is the Python package at /root/reference/pkg/src/cachetune
 * (cited as ct/<file>:<line>).  The ctypes binding a maintainer adds to the
 * reference is shown in INTEGRATION.md; the repo's own binding is
 * paper_2605_24022_b200/_lib.py.
 *
 * Conventions (all entry points):
 *   - return an int status (ct_status); 0 = OK.  ct_last_error() copies the
 *     message of the calling thread's last failure.  The Python shim maps
 *     statuses onto ct/errors.py:4-37 (ShapeError, InvalidParam, InvalidPlan,
 *     IoError).
 *   - tensors are caller-allocated device pointers (pinned host where said)
 *     with explicit int64 sizes/strides in ELEMENTS; nothing here allocates or
 *     frees caller memory.  Workspace is caller-provided, sized by the
 *     matching *_workspace_bytes() query.
 *   - every call takes a cudaStream_t (passed as void*), is asynchronous and
 *     never synchronises the device.
 *   - reentrant: no mutable globals except the per-thread error string and
 *     the atomic launch counters (ct_launch_stats).
 *   - token-major KV layout [token][head][dim] (ct/kvcore.py:31-66).
 */
#ifndef CACHETUNE_B200_H
#define CACHETUNE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CT_OK = 0,
  CT_ERR_SHAPE = 1,       /* ct/errors.py:8  ShapeError   */
  CT_ERR_PARAM = 2,       /* ct/errors.py:12 InvalidParam */
  CT_ERR_PLAN = 3,        /* ct/errors.py:16 InvalidPlan  */
  CT_ERR_IO = 4,          /* ct/errors.py:28 IoError      */
  CT_ERR_CUDA = 5,        /* CUDA runtime failure          */
  CT_ERR_UNSUPPORTED = 6  /* geometry this build does not handle */
} ct_status;

typedef enum { CT_F32 = 0, CT_BF16 = 1, CT_F64 = 2 } ct_dtype;

/* RoPE pairing, ct/rope.py:20-40 */
typedef enum { CT_ROPE_ADJACENT = 0, CT_ROPE_SPLIT = 1 } ct_rope_pairing;

int ct_version(void);
int ct_last_error(char* buf, size_t len);
/* number of SMs of the current device (0 without a device) */
int ct_device_sm_count(void);

/* Launch evidence: "kernel=count;kernel=count;..." for every kernel this
 * library launched successfully since load (or the last reset), e.g.
 * "attention_pp_kernel=31" proves the tcgen05 attention ran.  Host-side
 * counters only (no device sync). */
int ct_launch_stats(char* buf, size_t len);
void ct_launch_stats_reset(void);

/* ------------------------------------------------------------------ */
/* (1) frequency-domain scorer -- replaces ct/spectral.py:69-90
 * (_band_scores/low_freq_scores) and ct/spectral.py:149-159 (rank_chunk).
 *
 * Scores C chunks of equal geometry [L][N][H*D] in one call.  keys/values
 * element (c, l, n, lane) lives at base + c*ld_chunk + l*ld_layer + n*ld_token
 * + lane.  alpha in [0,1]; cutoff c = floor(alpha*(N/2+1)) is computed by the
 * caller exactly as ct/spectral.py:57-58 and passed as `cutoff`.
 * precision: CT_F64 (exact mode, float64 FFT like pocketfft) or CT_F32.
 * Outputs (device, may be NULL where marked):
 *   layer_scores [C][L][N] f64, agg_scores [C][N] f64 (sequential layer sum / L,
 *   ct/spectral.py:156), layer_order [C][L][N] int32 (nullable),
 *   agg_order [C][N] int32: stable descending order (ties -> lower index),
 *   ct/spectral.py:99-101. */
size_t ct_score_workspace_bytes(int64_t C, int64_t L, int64_t N, int64_t lanes,
                                int precision);
int ct_score_chunks(const void* keys, const void* values, int dtype,
                    int64_t C, int64_t L, int64_t N, int64_t lanes,
                    int64_t ld_token, int64_t ld_layer, int64_t ld_chunk,
                    int64_t cutoff, int precision,
                    double* layer_scores, double* agg_scores,
                    int32_t* layer_order, int32_t* agg_order,
                    void* workspace, size_t workspace_bytes, void* stream);

/* Same as ct_score_chunks with a band selector: band 0 = the low band above,
 * band 1 = the complementary high band (min(k, N-k) >= cutoff), the score the
 * reference's "highfreq" selection strategy uses
 * (ct/toymodel.py:355-358 -> ct/spectral.py high_freq_scores). */
int ct_score_chunks_band(const void* keys, const void* values, int dtype,
                         int64_t C, int64_t L, int64_t N, int64_t lanes,
                         int64_t ld_token, int64_t ld_layer, int64_t ld_chunk,
                         int64_t cutoff, int precision, int band,
                         double* layer_scores, double* agg_scores,
                         int32_t* layer_order, int32_t* agg_order,
                         void* workspace, size_t workspace_bytes, void* stream);

/* Single-chunk form of ct_score_chunks (the reference's rank_chunk /
 * low_freq_scores, ct/spectral.py:82-90,149-159): one chunk of L layers laid
 * out [L][N][ld_token] with lanes = H*D, exact (f64) mode, cutoff computed
 * here as floor(alpha * (N/2 + 1)) (ct/spectral.py:57-58).  alpha outside
 * [0,1] -> CT_ERR_PARAM before any work.  layer_scores [L][N] f64,
 * agg_scores [N] f64, agg_order [N] int32 (stable descending). */
int ct_score_chunk(const void* keys, const void* values, int dtype,
                   int64_t L, int64_t N, int64_t H, int64_t D, int64_t ld_token,
                   double alpha, double* layer_scores, double* agg_scores,
                   int32_t* agg_order, void* workspace, size_t workspace_bytes,
                   void* stream);

/* Fast scorer with a certified selection boundary (N = 2048, lanes a
 * multiple of 128; other geometries return CT_ERR_UNSUPPORTED and the caller
 * uses ct_score_chunks).  The aggregate scores of ct/spectral.py:149-159 are
 * computed with single-precision FFTs (relative error bound `guard`, see
 * DESIGN.md); agg_order [C][N] is their stable descending order with the
 * boundary between positions k-1 and k made exact: when the k-th and
 * (k+1)-th scores are within the guard, every token whose score could cross
 * the boundary is re-scored in float64 (direct projection, all layers) and
 * that window re-ordered, so agg_order[0..k) is the float64 top-k set
 * (ct/spectral.py:162-178).  wcount [C] (device int32): 0 = boundary
 * certified by the guard, w in (0, 64] = w tokens re-scored exactly,
 * w > 64 = window too wide, the caller must re-score the chunk with
 * ct_score_chunks (exact mode).  layer_scores [C][L][N] f64 (nullable) and
 * agg_scores [C][N] f64 are the single-precision-derived scores (window
 * tokens carry their float64 aggregate).  Asynchronous, no host sync.
 * band 0 = low band (default), 1 = high band. */
size_t ct_score_fast_workspace_bytes(int64_t C, int64_t L, int64_t N, int64_t lanes);
int ct_score_select_fast(const void* keys, const void* values, int dtype,
                         int64_t C, int64_t L, int64_t N, int64_t lanes,
                         int64_t ld_token, int64_t ld_layer, int64_t ld_chunk,
                         int64_t cutoff, int band, int64_t k, double guard,
                         double* layer_scores, double* agg_scores,
                         int32_t* agg_order, int32_t* wcount, void* workspace,
                         size_t workspace_bytes, void* stream);

/* Stable descending argsort of `rows` rows of n f64 scores (ties -> lower
 * index): ct/spectral.py:99-101.  order is int32 [rows][n]. */
int ct_desc_order(const double* scores, int64_t rows, int64_t n,
                  int32_t* order, void* stream);

/* ------------------------------------------------------------------ */
/* selection plan -- replaces ct/spectral.py:162-184 (indices_for_ratio /
 * complement_for_ratio) and the global assembly of ct/toymodel.py:246-267.
 * For chunk j (tokens [offsets[j], offsets[j+1]) on the global axis) the
 * first ks[j] entries of its aggregate order are recomputed.  Outputs
 * (device int32): rec_global ascending [sum k], keep_global ascending
 * [sum (N_j-k_j)], keep_src_row [sum(N_j-k_j)] = importance rank of each keep
 * token (its row in an importance-ordered pool).  offsets/ks/rec_base/
 * keep_base are DEVICE int64 arrays of n_chunks(+1) entries. */
/* One chunk's selection at ratio r -- selection_count / indices_for_ratio /
 * complement_for_ratio (ct/spectral.py:162-184): k = min(max(ceil(r*n -
 * 1e-9), 0), n) computed on the host (written to *k_out when non-NULL);
 * sel [k] = order[0..k) ascending, keep [n-k] = order[k..n) ascending (device
 * int32, chunk-local ids).  r outside [0,1] -> CT_ERR_PARAM before any work. */
int ct_select(const int32_t* order, int64_t n, double r, int32_t* sel,
              int32_t* keep, int64_t* k_out, void* stream);

int ct_selection_plan(const int32_t* agg_orders, const int64_t* offsets,
                      const int64_t* ks, const int64_t* rec_base,
                      const int64_t* keep_base, int64_t n_chunks,
                      int64_t max_chunk_tokens, int32_t* rec_global,
                      int32_t* keep_global, int32_t* keep_src_row,
                      void* stream);

/* ------------------------------------------------------------------ */
/* (3) deferred RoPE -- ct/rope.py:42-81.
 * Table of (cos, sin) for positions [0, n_pos) and pairs j < D/2:
 * angle = (p*scaling) * freqs[j] in float64 (freqs computed by the caller as
 * base**(-2j/D), ct/rope.py:42-44), cos/sin in float64.  Written as
 * double2 (table_f64, nullable) and/or float2 (table_f32, nullable),
 * layout [n_pos][D/2].  With `positions` (device int64 [n_pos], nullable)
 * row t holds the angles of position positions[t] (any sign) instead of t. */
int ct_rope_table(const double* freqs, int64_t half_dim, int64_t n_pos,
                  double scaling, const int64_t* positions, void* table_f64,
                  void* table_f32, void* stream);

/* Rotate rows: out[i] = rope(x[i], positions[i]) (ct/rope.py:75-81).
 * x/out [n][H][D] of dtype; f32/bf16 in; math in f64 for CT_F32 (bit-exact
 * formula of ct/rope.py:61-62), f32 for CT_BF16; CT_F64 rows in and out are
 * ct/rope.py:47-72 rope_rotate (f64 table required). */
int ct_rope_apply(const void* x, const int32_t* positions, int64_t n,
                  int64_t H, int64_t D, int dtype, int pairing,
                  const void* table, void* out, void* stream);

/* One reused segment of the blended cache (a chunk's keep rows for one
 * layer).  Row i of the segment holds local token tok[i] (tok: device int32);
 * it lands at global row pos0 + tok[i], K rotated by that global position
 * (deferred RoPE, ct/pipesim.py:346-351).  Source row: k/v + i*src_row_stride
 * when src_by_tok == 0 (an importance-ordered pool / staging buffer whose keep
 * set is a contiguous tail), k/v + tok[i]*src_row_stride when src_by_tok == 1
 * (a token-ordered chunk resident in HBM). */
typedef struct {
  const void* k;
  const void* v;
  const int32_t* tok;
  int64_t rows;
  int64_t pos0;
  int64_t src_by_tok;
} ct_segment;

#define CT_MAX_SEGMENTS 64

/* (2)+(3) fused sparse gather + deferred RoPE + blend -- replaces the
 * reuse half of ct/pipesim.py:322-357 (fuse_layer) and the in-path gather of
 * ct/toymodel.py:269-283.  segs is a HOST array (copied into the launch);
 * k_cache/v_cache [n_ctx][H][D] (cache_row_stride elements per row). */
int ct_gather_rope_blend(const ct_segment* segs, int n_segs, int64_t src_row_stride,
                         int64_t H, int64_t D, int dtype, int pairing,
                         const void* table, void* k_cache, void* v_cache,
                         int64_t cache_row_stride, void* stream);

/* (4, epilogue) QKV rope + scatter -- ct/toymodel.py:157-172.
 * qkv [A][ld_qkv] holds q (Hq*D) | k (Hkv*D) | v (Hkv*D) of dtype in_dtype.
 * Writes q_out [A][Hq][D] (q_dtype), rotated k and raw v into the caches at
 * rows positions[a], and optionally the pre-RoPE k into k_raw_out [A][Hkv][D]
 * (cache dtype).  Rotation math as ct_rope_apply. */
int ct_qkv_rope_scatter(const void* qkv, int64_t ld_qkv, int in_dtype,
                        const int32_t* positions, int64_t A, int64_t Hq,
                        int64_t Hkv, int64_t D, int pairing, const void* table,
                        void* q_out, int q_dtype, void* k_cache, void* v_cache,
                        int cache_dtype, int64_t cache_row_stride,
                        void* k_raw_out, void* stream);

/* Row scatter/gather (ct/kvcore.py:161-194): dst[idx[i]] = src[i] (scatter)
 * or dst[i] = src[idx[i]] (gather); row_bytes multiple of 4. */
int ct_scatter_rows(const void* src, const int32_t* idx, int64_t n,
                    int64_t row_bytes, void* dst, void* stream);
int ct_gather_rows(const void* src, const int32_t* idx, int64_t n,
                   int64_t row_bytes, void* dst, void* stream);


/* Importance-ordered pool image, the offline stage's last step (layout of
 * pool.py; replaces the reference's per-token CTKV writes,
 * ct/cachepool.py:167-230 + the keep-set ranges of :409-435):
 *   dst[((c*L + l)*N + p)*2 + side] (row_bytes each) =
 *       (side ? values : keys)[c*ld_chunk + l*ld_layer + order[c*N + p]*ld_token]
 * Strides in BYTES, multiples of 4 (16-byte rows and strides take the
 * vector path).  One launch for all C chunks. */
int ct_pool_permute(const void* keys, const void* values, int C, int L, int N,
                    int64_t ld_token, int64_t ld_layer, int64_t ld_chunk,
                    int64_t row_bytes, const int32_t* order, void* dst, void* stream);

/* ------------------------------------------------------------------ */
/* (4) selective-recompute attention -- ct/toymodel.py:176-183.
 * Queries q [A][Hq][D] at global positions q_pos[a] (ascending not
 * required); keys/values = the full blended cache [n_ctx][Hkv][D]; key j is
 * visible to query a iff j <= q_pos[a]; GQA: q-head h reads kv-head
 * h / (Hq/Hkv).  out [A][Hq][D] (out_dtype).  probs (nullable, f32
 * [Hq][A][n_ctx]) receives the normalised attention matrix (AttentionRecord,
 * ct/toymodel.py:92-110).
 * dtype CT_F32: SIMT fp32 path (1e-5 mode).  dtype CT_BF16: tcgen05/TMEM
 * path on sm_100a (bf16 operands, fp32 accumulation), D == 128.
 * A * (Hq/Hkv) <= 8 rows without probs (e.g. a first-token row alone): the
 * split-key path (key range split over ~2 CTAs per SM, fixed-order combine);
 * it needs ct_attention_workspace_bytes(...) of workspace (0 otherwise) and
 * returns CT_ERR_PARAM when the workspace is missing or short. */
size_t ct_attention_workspace_bytes(int64_t A, int64_t Hq, int64_t n_ctx,
                                    int64_t Hkv, int64_t D, int dtype);
int ct_selective_attention(const void* q, const int32_t* q_pos, int64_t A,
                           int64_t Hq, const void* k_cache, const void* v_cache,
                           int64_t n_ctx, int64_t Hkv, int64_t D,
                           int64_t cache_row_stride, double scale, int dtype,
                           void* out, int out_dtype, float* probs,
                           void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------------ */
/* transformer plumbing around the hot path (ct/toymodel.py:149,156,184-192) */

/* out[a] = table[tokens[a]] rows of `cols` f32 (embedding gather) */
int ct_embedding_gather(const float* table, const int32_t* tokens, int64_t A,
                        int64_t cols, float* out, void* stream);

/* h[a] += delta[a] (delta dtype, nullable); x[a] = h[a]/sqrt(mean(h^2)+eps)
 * written as x_dtype (ct/toymodel.py:88-89 with the residual add of :184). */
int ct_residual_rmsnorm(float* h, const void* delta, int delta_dtype, int64_t A,
                        int64_t cols, double eps, void* x_out, int x_dtype,
                        void* stream);

/* act[a][i] = f(gu[a][i], gu[a][inter+i]): SwiGLU silu(g)*u (kind 0) or
 * ReLU(g) (kind 1, ct/toymodel.py:186; then inter = cols). */
int ct_mlp_act(const void* gu, int64_t A, int64_t inter, int in_dtype,
               int kind, void* act, int act_dtype, void* stream);

/* act[m][i] = silu(g) * u with g = (x @ w)[m][i], u = (x @ w)[m][I + i]: the
 * SwiGLU gate/up projection and activation (ct/toymodel.py:186, w1 + act) in one
 * tcgen05 kernel (bf16 x [M][K] row stride ldx, w [K][2I] row stride ldw,
 * act [M][I] row stride ld_act; f32 accumulation, the [M][2I] product never
 * stored).  K % 64 == 0, I % 128 == 0, 16-byte aligned rows. */
int ct_gemm_swiglu(const void* x, int64_t M, int64_t K, int64_t ldx, const void* w,
                   int64_t I, int64_t ldw, void* act, int64_t ld_act, void* stream);

/* The dense projections of the bf16 step (ct/toymodel.py:157-159,184,186) on the
 * same CTA-pair tcgen05 GEMM: x bf16 [M][K] (row stride ldx) times w bf16
 * [K][N] (row stride ldw), f32 accumulation, and
 *   out_dtype CT_BF16, accumulate 0: out bf16 [M][N]  = x @ w   (QKV)
 *   out_dtype CT_F32,  accumulate 1: out f32  [M][N] += x @ w   (O- and
 *     down-projection into the f32 residual stream)
 * K % 64 == 0, N % 128 == 0, 16-byte aligned rows; other combinations
 * return CT_ERR_UNSUPPORTED.  Tiles are 256 x 256 per CTA pair, or 256 x 128
 * when that fills the last wave of tiles better. */
int ct_gemm_bf16(const void* x, int64_t M, int64_t K, int64_t ldx, const void* w, int64_t N,
                 int64_t ldw, void* out, int64_t ld_out, int out_dtype, int accumulate,
                 void* stream);

/* The q|k|v projection with the K4 epilogue (ct_qkv_rope_scatter) fused, for
 * the bf16 step with head_dim 128 and adjacent RoPE pairs
 * (ct/toymodel.py:157-163, ct/rope.py:40-70): qkv = x @ w (w bf16
 * [K][(Hq + 2 Hkv) 128], row stride ldw) in f32 accumulators, then q heads
 * rotated at positions[m] -> q_out bf16 [M][Hq][128]; k heads rotated ->
 * k_cache row positions[m]; v heads -> v_cache row positions[m] (row stride
 * cache_row_stride elements).  table = the f32 (cos, sin) pair table
 * [n_ctx][64] of ct_rope_table.  The [M][N] product never reaches HBM.
 * K % 64 == 0, Hq + 2 Hkv even, 16-byte aligned rows; D != 128 returns
 * CT_ERR_UNSUPPORTED. */
int ct_gemm_qkv_rope(const void* x, int64_t M, int64_t K, int64_t ldx, const void* w,
                     int64_t ldw, const int32_t* positions, const void* table, int64_t Hq,
                     int64_t Hkv, int64_t D, void* q_out, void* k_cache, void* v_cache,
                     int64_t cache_row_stride, void* stream);

/* ------------------------------------------------------------------ */
/* (2) sparse pinned-host -> HBM transfer on the copy engines
 * (ct/cachepool.py:409-481 with an importance-ordered pool so each
 * (chunk, layer) keep set is ONE contiguous tail).  Issues n cudaMemcpyAsync
 * host->device copies on `stream`. */
int ct_copy_ranges_h2d(void* const* dst, const void* const* src,
                       const int64_t* bytes, int64_t n, void* stream);

/* pinned host allocation helpers (cudaHostAlloc / cudaFreeHost) */
int ct_host_alloc(void** ptr, size_t bytes);
int ct_host_free(void* ptr);

#ifdef __cplusplus
}
#endif
#endif /* CACHETUNE_B200_H */
