"""The paper's offline stage on the GPU.

For each reusable chunk: isolated prefill at local positions producing the
pre-RoPE K/V (ct/toymodel.py:208-220, same kernels as the online path), the
frequency-domain ranking (ct/spectral.py:149-159, batched scorer), and the
importance-ordered pool write (pool.KvPool) the online sparse fetch reads as
one contiguous tail per (chunk, layer).  Optionally emits reference CTKV
files (ctkv.write_ctkv) so a reference deployment can consume the rankings.
"""

from __future__ import annotations

from pathlib import Path
from typing import Sequence

import torch

from .ctkv import write_ctkv
from .pool import KvPool
from .prefill import encode_chunk_isolated
from .spectral import rank_chunks


def prepare_pool(model, token_lists: Sequence, alpha: float = 0.5, precision: str = "f64",
                 location: str = "pinned", chunk_ids: Sequence[str] | None = None,
                 ctkv_dir: str | Path | None = None, timings: dict | None = None) -> KvPool:
    """Encode + rank + pool a set of chunks; returns the pool.  `timings`
    (optional dict) receives per-stage CUDA-event milliseconds."""
    ids = list(chunk_ids or [f"chunk{i}" for i in range(len(token_lists))])
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record()
    chunks = [encode_chunk_isolated(model, t, chunk_id=cid) for t, cid in zip(token_lists, ids)]
    ev[1].record()
    ranks = rank_chunks(chunks, alpha, precision)
    ev[2].record()
    pool = KvPool(chunks, ranks, location)
    ev[3].record()
    if ctkv_dir is not None:
        out = Path(ctkv_dir)
        out.mkdir(parents=True, exist_ok=True)
        for c, rk in zip(chunks, ranks):
            (out / f"{c.chunk_id}.ctkv").write_bytes(write_ctkv(c.to_host(), rk))
    if timings is not None:
        torch.cuda.synchronize()
        timings["encode_ms"] = ev[0].elapsed_time(ev[1])
        timings["rank_ms"] = ev[1].elapsed_time(ev[2])
        timings["pool_ms"] = ev[2].elapsed_time(ev[3])
    return pool
