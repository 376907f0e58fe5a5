"""Float64 oracle checks of a full-size request on sampled rows / heads
(the oracle cannot run a 32K/64K request end to end, so each
checked layer is compared piecewise against the reference arithmetic).

For a layer l of a finished `SelectivePrefillEngine` step:

* blend: the oracle's `fuse_layer` (ct/pipesim.py:322-357 -> ct/rope.py:75-81)
  rebuilds the whole blended cache of layer l from the pool's pre-RoPE keep
  rows (rotated in float64 at their global positions) and the engine's
  recomputed rows; the engine's cache must equal it within the tolerance;
* attention: for `rows` sampled query rows (the last suffix row always
  included) and two kv heads (their 2*G query heads), the oracle attention
  (ct/toymodel.py:176-183: scores / sqrt(D), key j visible iff j <= pos,
  float64 softmax, P V) over the engine's blended cache must match the
  engine's attention output rows.

Tolerance metric: max|got - want| / max|want| per tensor."""

from __future__ import annotations

import numpy as np
import torch

from oracle import cachetune_oracle as O


def snapshot_hook(eng, layers, rows):
    """hook for SelectivePrefillEngine.step: copies the rotated q rows and the
    attention output rows of `layers` after each of them ran."""
    snaps = {}
    idx = torch.as_tensor(np.asarray(rows, dtype=np.int64), device=eng.model.device)
    cfg = eng.model.config

    def hook(l, phase):
        if phase != "end" or l not in layers:
            return
        b = eng.buffers
        snaps[l] = {
            "q": b.q.index_select(0, idx).double().cpu().numpy(),
            "ctx": b.ctx.index_select(0, idx).double().cpu().numpy().reshape(
                len(rows), cfg.n_heads, cfg.head_dim),
        }
    return hook, snaps


def sample_rows(a: int, n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    rows = rng.choice(a - 1, size=min(n - 1, a - 1), replace=False)
    return np.sort(np.append(rows, a - 1))


def oracle_blend_error(eng, chunks, l: int) -> dict:
    """Normwise error of the engine's blended K/V of layer l vs O.fuse_layer."""
    cfg = eng.model.config
    n = eng.n_ctx
    keep = eng.keep.long().cpu().numpy()
    pos = eng.positions.long().cpu().numpy()
    N = eng.pool.N
    ci, tok = keep // N, keep % N
    k_raw = np.empty((keep.size, cfg.kv_heads, cfg.head_dim), dtype=np.float32)
    v_raw = np.empty_like(k_raw)
    for c in np.unique(ci):
        m = ci == c
        t = torch.as_tensor(tok[m], device=eng.model.device)
        ch = chunks[eng.chunk_ids[int(c)]]
        k_raw[m] = ch.keys[l].index_select(0, t).float().cpu().numpy()
        v_raw[m] = ch.values[l].index_select(0, t).float().cpu().numpy()
    kc = eng.cache[l, 0].float().cpu().numpy()
    vc = eng.cache[l, 1].float().cpu().numpy()
    rp = cfg.rope_params
    rope = O.Rope(rp.head_dim, rp.base, rp.scaling, rp.pairing)
    want_k, want_v = O.fuse_layer(k_raw, v_raw, keep, kc[pos], vc[pos], pos, keep, rope, n)
    return {"k": O.normwise_rel(kc, want_k), "v": O.normwise_rel(vc, want_v),
            "k_reused": O.normwise_rel(kc[keep], want_k[keep])}


def oracle_attention_error(eng, snap: dict, rows: np.ndarray, kv_heads=(0, 5)) -> float:
    """Normwise error of the engine's attention rows vs the float64 oracle on
    the engine's own blended cache, for the q heads of `kv_heads`."""
    cfg = eng.model.config
    G = cfg.n_heads // cfg.kv_heads
    l_cache = snap["layer"]
    kc = eng.cache[l_cache, 0].double().cpu().numpy()
    vc = eng.cache[l_cache, 1].double().cpu().numpy()
    pos = eng.positions.long().cpu().numpy()[rows]
    heads = [g * G + i for g in kv_heads for i in range(G)]
    q = snap["q"][:, heads, :]
    causal = np.arange(eng.n_ctx)[None, :] <= pos[:, None]
    want, _ = O._attention(q, kc[:, list(kv_heads), :], vc[:, list(kv_heads), :], causal,
                           len(heads), len(kv_heads), cfg.head_dim, False)
    got = snap["ctx"][:, heads, :]
    return O.normwise_rel(got, want)


def check_request(eng, chunks, suffix, layers, n_rows=64, seed=0, tol_attn=2e-2,
                  tol_blend=2e-2):
    """Run one step with snapshots and check `layers` against the oracle.
    Returns {layer: {"blend": ..., "attention": ...}} (errors)."""
    rows = sample_rows(eng.A, n_rows, seed)
    hook, snaps = snapshot_hook(eng, set(layers), rows)
    eng.step(suffix, hook=hook)
    torch.cuda.synchronize()
    out = {}
    last = eng.model.config.n_layers - 1
    for l in layers:
        snap = dict(snaps[l], layer=l)
        r = rows
        if l == last:  # the last layer runs attention on the first-token row only
            sel = np.flatnonzero(rows == eng.A - 1)
            snap = {"q": snap["q"][sel], "ctx": snap["ctx"][sel], "layer": l}
            r = rows[sel]
        att = oracle_attention_error(eng, snap, r)
        blend = oracle_blend_error(eng, chunks, l)
        out[l] = {"attention": att, **{f"blend_{k}": v for k, v in blend.items()}}
        assert att <= tol_attn, (l, out[l])
        assert max(blend.values()) <= tol_blend, (l, out[l])
    return out
