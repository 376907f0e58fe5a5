"""CPU oracle for the CacheTune online selective-recompute prefill path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package
(`paper_2605_24022_b200/`) may import, call or link this module.  Only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs use it, and only as the checker / the CPU arm.

This is a numpy restatement of the reference algorithm (references are to
`/root/reference/pkg/src/cachetune/`, written `ct/<file>:<line>`).  The
reference itself is pure Python/numpy; its only third-party arithmetic on
this path is numpy's pocketfft (`numpy.fft.rfft/irfft`, numpy 2.3.5 in this
image, pyproject pins only `numpy>=1.24`) and OpenBLAS for matmuls.  The
restatement uses the same numpy calls for the FFT so the float64 scores are
the reference's own arithmetic.

Parity pin: `tests/golden/make_golden.py` imports the live reference in the
build container and writes its outputs to `tests/golden/*.npz`;
`tests/test_oracle_golden.py` checks this module against every fixture
(bit-exact orders / index sets, float tensors to 1e-12).

Extensions beyond the reference toy model (needed for the Llama-3-8B /
Mistral-7B geometries of BASELINE.json configs 2-5; the reference is MHA with
an optional ReLU MLP only, ct/toymodel.py:73-77):
  * n_kv_heads < n_heads (GQA): wk/wv are hid x (n_kv_heads*D); q-head h reads
    kv-head h // (n_heads // n_kv_heads).
  * mlp="swiglu": h += (silu(x Wg) * (x Wu)) Wd with x = rms_norm(h).
  * rope pairing / base / scaling are exposed (ct/rope.py:20-44).
With n_kv_heads == n_heads and mlp in (False, "relu") the restatement draws
the same weights in the same order as ct/toymodel.py:61-79 and is validated
against the reference to <= 1e-12 (tests/test_oracle_golden.py).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

NORM_EPS = 1e-6  # ct/toymodel.py:28


# ---------------------------------------------------------------------------
# spectral scoring and selection (ct/spectral.py)

def cutoff_index(alpha: float, n_freqs: int) -> int:
    """ct/spectral.py:57-58 -- c = floor(alpha * n_freqs) as a float product."""
    return int(math.floor(alpha * n_freqs))


def low_freq_scores(keys: np.ndarray, values: np.ndarray,
                    alpha: float = 0.5, band: str = "low") -> np.ndarray:
    """ct/spectral.py:69-90 (_band_scores, band='low').

    keys/values: [N, H, D] float32 (token-major).  For each tensor: float64
    rfft along tokens, zero bins >= c (band='high': bins < c, ct/spectral.py:47-54),
    irfft(n=N), per-token L2 norm over the flattened H*D row;
    score = 0 + 0.5*|K~_i| + 0.5*|V~_i|.
    """
    if keys.shape != values.shape:
        raise ValueError("shape mismatch")
    if not 0.0 <= alpha <= 1.0:
        raise ValueError("alpha out of range")
    n = keys.shape[0]
    out = np.zeros(n, dtype=np.float64)
    for t in (keys, values):
        spec = np.fft.rfft(np.asarray(t, dtype=np.float32).astype(np.float64), axis=0)
        c = cutoff_index(alpha, spec.shape[0])
        if band == "low":
            spec[c:] = 0.0
        else:
            spec[:c] = 0.0
        recon = np.fft.irfft(spec, n=n, axis=0)
        out += 0.5 * np.linalg.norm(recon.reshape(n, -1), axis=1)
    return out


def high_freq_scores(keys: np.ndarray, values: np.ndarray, alpha: float = 0.5) -> np.ndarray:
    """ct/spectral.py:93-96 -- the complementary high band."""
    return low_freq_scores(keys, values, alpha, band="high")


def descending_order(scores: np.ndarray) -> np.ndarray:
    """ct/spectral.py:99-101 -- stable argsort of -scores (ties -> lower index)."""
    return np.argsort(-scores, kind="stable").astype(np.int64)


def rank_chunk(keys_layers, values_layers, alpha: float = 0.5):
    """ct/spectral.py:149-159.  Returns (scores[L,N] f64, per_layer_order[L,N],
    aggregate_order[N]); aggregate = stable desc order of scores.mean(axis=0)."""
    scores = np.stack([low_freq_scores(k, v, alpha)
                       for k, v in zip(keys_layers, values_layers)])
    orders = np.stack([descending_order(row) for row in scores])
    agg = descending_order(scores.mean(axis=0))
    return scores, orders, agg


def selection_count(r: float, n_tokens: int) -> int:
    """ct/spectral.py:162-172 -- min(max(ceil(r*N - 1e-9), 0), N)."""
    if not 0.0 <= r <= 1.0:
        raise ValueError("ratio out of range")
    k = math.ceil(r * n_tokens - 1e-9)
    return min(max(k, 0), n_tokens)


def indices_for_ratio(aggregate_order: np.ndarray, r: float) -> np.ndarray:
    """ct/spectral.py:175-178."""
    k = selection_count(r, aggregate_order.size)
    return np.sort(aggregate_order[:k])


def complement_for_ratio(aggregate_order: np.ndarray, r: float) -> np.ndarray:
    """ct/spectral.py:181-184."""
    k = selection_count(r, aggregate_order.size)
    return np.sort(aggregate_order[k:])


# ---------------------------------------------------------------------------
# deferred RoPE (ct/rope.py)

@dataclass(frozen=True)
class Rope:
    head_dim: int
    base: float = 10000.0
    scaling: float = 1.0
    pairing: str = "adjacent"

    def freqs(self) -> np.ndarray:
        """ct/rope.py:42-44 -- base ** (-2 j / D), float64."""
        j = np.arange(self.head_dim // 2, dtype=np.float64)
        return self.base ** (-2.0 * j / self.head_dim)


def rope_rotate(x: np.ndarray, positions: np.ndarray, rope: Rope) -> np.ndarray:
    """ct/rope.py:47-72 -- float64 rotation of [N, H, D] at given positions."""
    n, _, d = x.shape
    angles = np.outer(np.asarray(positions).astype(np.float64) * rope.scaling,
                      rope.freqs())
    cos = np.cos(angles)[:, None, :]
    sin = np.sin(angles)[:, None, :]
    x = x.astype(np.float64)
    if rope.pairing == "adjacent":
        a, b = x[..., 0::2], x[..., 1::2]
    else:
        a, b = x[..., : d // 2], x[..., d // 2:]
    ra = a * cos - b * sin
    rb = a * sin + b * cos
    out = np.empty_like(x)
    if rope.pairing == "adjacent":
        out[..., 0::2] = ra
        out[..., 1::2] = rb
    else:
        out[..., : d // 2] = ra
        out[..., d // 2:] = rb
    return out


def rope_apply(keys: np.ndarray, positions, rope: Rope) -> np.ndarray:
    """ct/rope.py:75-81 -- rotate in float64, store float32."""
    return rope_rotate(np.asarray(keys, dtype=np.float32), np.asarray(positions),
                       rope).astype(np.float32)


# ---------------------------------------------------------------------------
# scatter fusion (ct/pipesim.py:322-357, ct/kvcore.py:171-194)

def fuse_layer(k_reuse, v_reuse, keep_idx, k_new, v_new, rec_idx,
               positions, rope: Rope, n: int):
    """ct/pipesim.py:322-357: partition check, NaN buffers, reused K rotated
    at `positions`, recomputed rows scattered verbatim."""
    keep = np.asarray(keep_idx, dtype=np.int64)
    rec = np.asarray(rec_idx, dtype=np.int64)
    merged = np.concatenate([keep, rec])
    if merged.size != n or not np.array_equal(np.sort(merged), np.arange(n)):
        raise ValueError("keep/recompute sets must partition [0, n)")
    ref = k_reuse if k_reuse is not None else k_new
    h, d = ref.shape[1], ref.shape[2]
    k_buf = np.full((n, h, d), np.nan, dtype=np.float32)
    v_buf = np.full((n, h, d), np.nan, dtype=np.float32)
    if keep.size:
        k_buf[keep] = rope_apply(k_reuse, positions, rope)
        v_buf[keep] = np.asarray(v_reuse, dtype=np.float32)
    if rec.size:
        k_buf[rec] = k_new
        v_buf[rec] = v_new
    return k_buf, v_buf


# ---------------------------------------------------------------------------
# toy transformer, restated with GQA / SwiGLU extensions (ct/toymodel.py)

@dataclass(frozen=True)
class ModelConfig:
    """ct/toymodel.py:31-55 plus n_kv_heads / mlp kind / rope knobs."""
    seed: int = 0
    n_layers: int = 4
    n_heads: int = 2
    head_dim: int = 8
    vocab_size: int = 256
    mlp: object = False            # False | "relu" (ref mlp=True) | "swiglu"
    rope_base: float = 10000.0
    n_kv_heads: int | None = None
    intermediate: int | None = None  # swiglu width (default 4*hid)
    rope_pairing: str = "adjacent"
    rope_scaling: float = 1.0

    @property
    def hidden_dim(self) -> int:
        return self.n_heads * self.head_dim

    @property
    def kv_heads(self) -> int:
        return self.n_kv_heads or self.n_heads

    @property
    def mlp_kind(self):
        if self.mlp is True:
            return "relu"
        return self.mlp or None

    @property
    def rope(self) -> Rope:
        return Rope(self.head_dim, self.rope_base, self.rope_scaling,
                    self.rope_pairing)


class Model:
    """Weights drawn like ct/toymodel.py:61-79: default_rng(seed), U(-1,1)/sqrt(hid),
    in order embedding, per layer (wq, wk, wv, wo, [mlp...]), w_out."""

    def __init__(self, config: ModelConfig, weights: dict | None = None):
        self.config = config
        if weights is not None:
            self.embedding = weights["embedding"]
            self.layers = weights["layers"]
            self.w_out = weights["w_out"]
            return
        hid = config.hidden_dim
        kvd = config.kv_heads * config.head_dim
        rng = np.random.default_rng(config.seed)
        scale = 1.0 / np.sqrt(hid)

        def w(*shape):
            return rng.uniform(-1.0, 1.0, size=shape) * scale

        self.embedding = w(config.vocab_size, hid)
        self.layers = []
        for _ in range(config.n_layers):
            layer = {"wq": w(hid, hid), "wk": w(hid, kvd),
                     "wv": w(hid, kvd), "wo": w(hid, hid)}
            if config.mlp_kind == "relu":
                layer["w1"] = w(hid, 4 * hid)
                layer["w2"] = w(4 * hid, hid)
            elif config.mlp_kind == "swiglu":
                inter = config.intermediate or 4 * hid
                layer["wg"] = w(hid, inter)
                layer["wu"] = w(hid, inter)
                layer["wd"] = w(inter, hid)
            self.layers.append(layer)
        self.w_out = w(hid, config.vocab_size)


def rms_norm(x: np.ndarray) -> np.ndarray:
    """ct/toymodel.py:88-89 (no weight)."""
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + NORM_EPS)


def _attention(q_rot, k_ctx, v_ctx, causal, n_heads, n_kv, d, want_probs):
    """ct/toymodel.py:176-183 with GQA head mapping; matmul per kv group."""
    a = q_rot.shape[0]
    group = n_heads // n_kv
    ctx = np.empty((a, n_heads, d))
    probs = np.empty((n_heads, a, k_ctx.shape[0])) if want_probs else None
    inv = 1.0 / np.sqrt(d)
    for h in range(n_heads):
        g = h // group
        s = (q_rot[:, h, :] @ k_ctx[:, g, :].T) * inv
        s = np.where(causal, s, -np.inf)
        s -= s.max(axis=-1, keepdims=True)
        p = np.exp(s)
        p /= p.sum(axis=-1, keepdims=True)
        ctx[:, h, :] = p @ v_ctx[:, g, :]
        if want_probs:
            probs[h] = p
    return ctx, probs


def run(model: Model, tokens, positions, reused_per_layer=None,
        n_context=None, want_probs=True, logits_rows="all"):
    """ct/toymodel.py:135-193 (shared forward engine)."""
    cfg = model.config
    hid, nh, nkv, d = cfg.hidden_dim, cfg.n_heads, cfg.kv_heads, cfg.head_dim
    tokens = np.asarray(tokens, dtype=np.int64)
    positions = np.asarray(positions, dtype=np.int64)
    a = tokens.size
    if n_context is None:
        n_context = a
    h = model.embedding[tokens]
    kv_out, k_raw_out, attn_out = [], [], []
    col_positions = positions if reused_per_layer is None else np.arange(n_context)
    causal = col_positions[None, :] <= positions[:, None]
    for l, layer in enumerate(model.layers):
        x = rms_norm(h)
        q = (x @ layer["wq"]).reshape(a, nh, d)
        k_raw = (x @ layer["wk"]).reshape(a, nkv, d)
        v = (x @ layer["wv"]).reshape(a, nkv, d)
        q_rot = rope_rotate(q, positions, cfg.rope)
        k_rot = rope_rotate(k_raw, positions, cfg.rope)
        if reused_per_layer is None:
            k_ctx, v_ctx = k_rot, v
        else:
            k_keep, v_keep, keep_global = reused_per_layer[l]
            k_full, v_full = fuse_layer(k_keep, v_keep, keep_global,
                                        k_rot.astype(np.float32),
                                        v.astype(np.float32), positions,
                                        keep_global, cfg.rope, n_context)
            k_ctx = k_full.astype(np.float64)
            v_ctx = v_full.astype(np.float64)
        ctx, probs = _attention(q_rot, k_ctx, v_ctx, causal, nh, nkv, d, want_probs)
        attn_out.append(probs)
        h = h + ctx.reshape(a, hid) @ layer["wo"]
        if cfg.mlp_kind == "relu":
            h = h + np.maximum(rms_norm(h) @ layer["w1"], 0.0) @ layer["w2"]
        elif cfg.mlp_kind == "swiglu":
            xm = rms_norm(h)
            g = xm @ layer["wg"]
            h = h + ((g / (1.0 + np.exp(-g))) * (xm @ layer["wu"])) @ layer["wd"]
        k_raw_out.append(k_raw)
        kv_out.append((k_ctx.astype(np.float32), v_ctx.astype(np.float32)))
    if logits_rows == "last":
        logits = h[-1:] @ model.w_out
    else:
        logits = h @ model.w_out
    return h, kv_out, k_raw_out, attn_out, logits


def full_prefill(model: Model, tokens, **kw):
    """ct/toymodel.py:196-205 -> (kv per layer (K post-RoPE f32, V f32), probs, logits)."""
    toks = np.asarray(tokens, dtype=np.int64)
    _, kv, _, attn, logits = run(model, toks, np.arange(toks.size), **kw)
    return kv, attn, logits


def encode_chunk_isolated(model: Model, tokens):
    """ct/toymodel.py:208-220 -> (keys_raw [L][N,Hkv,D] f32, values [L] f32)."""
    toks = np.asarray(tokens, dtype=np.int64)
    _, kv, k_raw, _, _ = run(model, toks, np.arange(toks.size), want_probs=False)
    return ([k.astype(np.float32) for k in k_raw], [v for _, v in kv])


def selective_prefill(model: Model, chunks, aggregate_orders, suffix_tokens, r,
                      **kw):
    """ct/toymodel.py:223-311.

    chunks: list of (keys_raw [L] arrays, values [L] arrays, source_tokens).
    Returns dict(kv, attention, logits, query_positions, rec_global, keep_global).
    """
    cfg = model.config
    sizes = [c[2].size for c in chunks]
    offsets = np.cumsum([0] + sizes)
    history = int(offsets[-1])
    suffix = np.asarray(suffix_tokens, dtype=np.int64)
    n_context = history + suffix.size
    rec_parts, keep_parts, tok_parts = [], [], []
    for (kr, vs, src), agg, off in zip(chunks, aggregate_orders, offsets):
        rec_local = indices_for_ratio(np.asarray(agg), r)
        keep_local = complement_for_ratio(np.asarray(agg), r)
        rec_parts.append(rec_local + off)
        keep_parts.append(keep_local + off)
        tok_parts.append(np.asarray(src)[rec_local])
    rec_global = np.concatenate(rec_parts).astype(np.int64)
    keep_global = np.concatenate(keep_parts).astype(np.int64)
    active_positions = np.concatenate([rec_global, np.arange(history, n_context)])
    active_tokens = np.concatenate(tok_parts + [suffix]).astype(np.int64)
    order = np.argsort(active_positions, kind="stable")
    active_positions = active_positions[order]
    active_tokens = active_tokens[order]
    reused = []
    for l in range(cfg.n_layers):
        if keep_global.size:
            keys = np.concatenate([np.asarray(c[0][l])[kp - off]
                                   for c, kp, off in zip(chunks, keep_parts, offsets)])
            vals = np.concatenate([np.asarray(c[1][l])[kp - off]
                                   for c, kp, off in zip(chunks, keep_parts, offsets)])
            reused.append((keys, vals, keep_global))
        else:
            reused.append((None, None, keep_global))
    if active_tokens.size == 0:
        kv = [fuse_layer(k, v, kg, None, None, np.empty(0, np.int64), kg,
                         cfg.rope, n_context) for k, v, kg in reused]
        return dict(kv=kv, attention=None, logits=np.zeros((0, cfg.vocab_size)),
                    query_positions=active_positions, rec_global=rec_global,
                    keep_global=keep_global)
    _, kv, _, attn, logits = run(model, active_tokens, active_positions,
                                 reused_per_layer=reused, n_context=n_context, **kw)
    return dict(kv=kv, attention=attn, logits=logits,
                query_positions=active_positions, rec_global=rec_global,
                keep_global=keep_global)


# ---------------------------------------------------------------------------
# synthetic inputs (pattern of ct/cli.py:55-64 and ct/toymodel.py:402-406)

def synthetic_chunk(seed: int, n_layers: int, n_tokens: int, n_heads: int,
                    head_dim: int):
    """Seeded N(0,1) float32 chunk: all key layers, then all value layers."""
    rng = np.random.default_rng(seed)
    keys = [rng.standard_normal((n_tokens, n_heads, head_dim)).astype(np.float32)
            for _ in range(n_layers)]
    vals = [rng.standard_normal((n_tokens, n_heads, head_dim)).astype(np.float32)
            for _ in range(n_layers)]
    return keys, vals


def normwise_rel(got, want) -> float:
    """max|got - want| / max|want|."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    den = float(np.max(np.abs(want))) if want.size else 0.0
    if den == 0.0:
        return float(np.max(np.abs(got))) if got.size else 0.0
    return float(np.max(np.abs(got - want)) / den)
