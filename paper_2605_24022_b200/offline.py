"""The paper's offline stage on the GPU.

For a set of reusable chunks:

1. encode: each chunk's isolated prefill at local positions
   (ct/toymodel.py:208-220, the online path's kernels) writes its pre-RoPE K
   and V straight into the scorer's batch layout [C, L, N, Hkv, D] -- no
   per-chunk staging, no stack copy;
2. rank: one scorer launch set over the whole batch (ct/spectral.py:149-159,
   `score_device`), aggregate orders left on the device;
3. pool: ONE `ct_pool_permute` launch writes the importance-ordered pool image
   (pool.KvPool layout) from the batch; a pinned pool then takes one D2H copy.

Optionally emits reference CTKV files (ctkv.write_ctkv) so a reference
deployment can consume the rankings.
"""

from __future__ import annotations

from pathlib import Path
from typing import Sequence

import numpy as np
import torch

from . import _dev
from .ctkv import write_ctkv
from .errors import InvalidParam
from .pool import KvPool
from .prefill import as_gpu_model, encode_chunk_isolated
from .spectral import DEFAULT_ALPHA, ImportanceRanking, score_device


def _batch_setup(model, token_lists, chunk_ids, out):
    g = as_gpu_model(model)
    if len(token_lists) == 0:
        raise InvalidParam("no chunks to encode")
    n = len(token_lists[0])
    if any(len(t) != n for t in token_lists):
        raise InvalidParam("offline batch chunks must have one token count")
    ids = list(chunk_ids or [f"chunk{i}" for i in range(len(token_lists))])
    if len(ids) != len(token_lists):
        raise InvalidParam("one chunk id per token list")
    cfg = g.config
    shape = (len(token_lists), cfg.n_layers, n, cfg.kv_heads, cfg.head_dim)
    if out is None:
        keys = torch.empty(shape, dtype=g.dtype, device=g.device)
        vals = torch.empty(shape, dtype=g.dtype, device=g.device)
    else:
        keys, vals = out
        if any(tuple(t.shape) != shape or t.dtype != g.dtype or not t.is_contiguous()
               for t in (keys, vals)):
            raise InvalidParam(f"out batch tensors must be contiguous {shape} {g.dtype}")
    return g, ids, keys, vals


def encode_batch(model, token_lists: Sequence, chunk_ids: Sequence[str] | None = None,
                 out=None):
    """Encode equal-length chunks into one [C, L, N, Hkv, D] K batch and V
    batch (`out`=(keys, values) to reuse buffers); returns (keys, values,
    [DeviceChunk views of the batch])."""
    g, ids, keys, vals = _batch_setup(model, token_lists, chunk_ids, out)
    chunks = [encode_chunk_isolated(g, t, chunk_id=cid, out=(keys[i], vals[i]))
              for i, (t, cid) in enumerate(zip(token_lists, ids))]
    return keys, vals, chunks


def encode_and_rank(model, token_lists: Sequence, alpha: float = DEFAULT_ALPHA,
                    precision: str = "f64", chunk_ids: Sequence[str] | None = None, out=None):
    """The offline stage with scoring overlapped with encoding: chunk c's
    scorer launch set runs on a side stream while chunk c+1 is encoded.  The
    scorer is FP-pipe bound (SIMT FFTs) and the encode is tensor-pipe bound
    (cuBLAS GEMMs + tcgen05 attention), so the two share the SMs instead of
    running back to back.  Returns (keys, values, chunks, scores) with
    `scores` the `score_device` dict of the whole batch; results are
    identical to encode_batch + score_device (the same launches per chunk)."""
    g, ids, keys, vals = _batch_setup(model, token_lists, chunk_ids, out)
    C, L, n = keys.shape[0], keys.shape[1], keys.shape[2]
    dev = keys.device
    scores = {"layer_scores": torch.empty((C, L, n), dtype=torch.float64, device=dev),
              "agg": torch.empty((C, n), dtype=torch.float64, device=dev),
              "agg_order": torch.empty((C, n), dtype=torch.int32, device=dev),
              "layer_order": torch.empty((C, L, n), dtype=torch.int32, device=dev)}
    main = torch.cuda.current_stream(dev)
    side = torch.cuda.Stream(device=dev)
    side.wait_stream(main)  # the batch tensors above were allocated on main
    chunks = []
    for i, (t, cid) in enumerate(zip(token_lists, ids)):
        chunks.append(encode_chunk_isolated(g, t, chunk_id=cid, out=(keys[i], vals[i])))
        done = torch.cuda.Event()
        done.record(main)
        side.wait_event(done)
        with torch.cuda.stream(side):
            score_device(keys[i:i + 1], vals[i:i + 1], alpha, precision,
                         want_layer_order=True,
                         out={k: v[i:i + 1] for k, v in scores.items()})
    main.wait_stream(side)
    return keys, vals, chunks, scores


def rankings_from_scores(out: dict, alpha: float) -> list:
    """ImportanceRanking per chunk from a `score_device` batch result taken
    with want_layer_order=True (the device aggregate orders stay attached for
    the pool)."""
    ls = out["layer_scores"].cpu().numpy()
    lo = out["layer_order"].cpu().numpy()
    ao = out["agg_order"].cpu().numpy()
    res = []
    for i in range(ao.shape[0]):
        n = ao.shape[1]
        res.append(ImportanceRanking(
            per_layer_scores=ls[i],
            per_layer_order=lo[i].astype(np.int64),
            aggregate_order=ao[i].astype(np.int64), alpha=alpha, n_tokens=n,
            device_aggregate=out["agg_order"][i]))
    return res


def prepare_pool(model, token_lists: Sequence, alpha: float = DEFAULT_ALPHA,
                 precision: str = "f64", location: str = "pinned",
                 chunk_ids: Sequence[str] | None = None, ctkv_dir: str | Path | None = None,
                 timings: dict | None = None, resident_layers: int = 0,
                 overlap: bool = True) -> KvPool:
    """Encode + rank + pool a set of equal-length chunks; returns the pool.
    overlap: score each chunk on a side stream while the next one is encoded
    (`encode_and_rank`); otherwise encode all, then score the batch.
    `timings` (optional dict) receives per-stage CUDA-event milliseconds
    (encode_ms -- encode and, with overlap, the overlapped scoring; rank_ms --
    the scoring left after the encode; pool_ms) and the permute launch count."""
    if location not in ("hbm", "pinned"):
        raise InvalidParam(f"unknown pool location {location!r}")
    _dev.require_cuda()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    if overlap:
        keys, vals, chunks, out = encode_and_rank(model, token_lists, alpha, precision,
                                                  chunk_ids)
        ev[1].record()
    else:
        keys, vals, chunks = encode_batch(model, token_lists, chunk_ids)
        ev[1].record()
        out = score_device(keys, vals, alpha, precision, want_layer_order=True)
    ev[2].record()
    ranks = rankings_from_scores(out, alpha)
    ev_pool = torch.cuda.Event(enable_timing=True)
    ev_pool.record()
    pool = KvPool(chunks, ranks, location, resident_layers=resident_layers)
    ev[3].record()
    if ctkv_dir is not None:
        dst = Path(ctkv_dir)
        dst.mkdir(parents=True, exist_ok=True)
        for c, rk in zip(chunks, ranks):
            (dst / f"{c.chunk_id}.ctkv").write_bytes(write_ctkv(c.to_host(), rk))
    if timings is not None:
        torch.cuda.synchronize()
        timings["chunks"] = len(chunks)
        timings["encode_ms"] = ev[0].elapsed_time(ev[1])
        timings["rank_ms"] = ev[1].elapsed_time(ev[2])
        timings["pool_ms"] = ev_pool.elapsed_time(ev[3])
        timings["permute_launches"] = pool.permute_launches
    return pool


__all__ = ["encode_and_rank", "encode_batch", "prepare_pool", "rankings_from_scores"]
