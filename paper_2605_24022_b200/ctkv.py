"""CTKV chunk files <-> the importance-ordered pool.

The reference serialises a chunk as (little-endian, ct/cachepool.py:10-21,
40-44, 167-230):

    magic "CTKV" | version u32 = 1 | L | N | H | D | dtype (0 = f32) |
    flags (bit0: keys are pre-RoPE)
    per layer: K rows [N][H][D] f32, then V rows f32
    optional ranking block: alpha f64 | per-layer orders L*N u32 |
    aggregate order N u32 | per-layer scores L*N f64

`write_ctkv` / `read_ctkv` reproduce that format byte for byte (host I/O).
`pool_from_ctkv` loads ranked CTKV files straight into a `KvPool`: the
token-order payload is uploaded once and permuted into importance order on
the device (ct_gather_rows), so the online sparse fetch stays one contiguous
tail per (chunk, layer); the byte accounting of `plan_sparse_fetch` is the
reference's (|keep| * H * D * dsize * 2).
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np
import torch

from .errors import InvalidPlan, IoError, ShapeError
from .kvcore import DeviceChunk, DtypeCode, KvChunk, SeqTensor
from .spectral import ImportanceRanking

MAGIC = b"CTKV"
VERSION = 1
HEADER = struct.Struct("<4s7I")
FLAG_PRE_ROPE = 1
DTYPE_SIZE = 4


def layer_bytes(n: int, h: int, d: int) -> int:
    return 2 * n * h * d * DTYPE_SIZE


def ranking_block_bytes(l: int, n: int) -> int:
    return 8 + l * n * 4 + n * 4 + l * n * 8


def chunk_file_bytes(l: int, n: int, h: int, d: int, with_ranking: bool) -> int:
    return HEADER.size + l * layer_bytes(n, h, d) + (ranking_block_bytes(l, n) if with_ranking else 0)


def write_ctkv(chunk, ranking=None) -> bytes:
    """Serialise a (reference or own) KvChunk and optional ranking."""
    keys = [np.asarray(k.data, dtype="<f4") for k in chunk.keys_raw]
    vals = [np.asarray(v.data, dtype="<f4") for v in chunk.values]
    l = len(keys)
    n, h, d = keys[0].shape
    parts = [HEADER.pack(MAGIC, VERSION, l, n, h, d, int(getattr(chunk, "dtype_code", 0)),
                         FLAG_PRE_ROPE)]
    for k, v in zip(keys, vals):
        parts += [k.tobytes(), v.tobytes()]
    if ranking is not None:
        if ranking.n_tokens != n or ranking.n_layers != l:
            raise ShapeError("ranking geometry disagrees with chunk")
        parts += [struct.pack("<d", ranking.alpha),
                  np.asarray(ranking.per_layer_order).astype("<u4").tobytes(),
                  np.asarray(ranking.aggregate_order).astype("<u4").tobytes(),
                  np.asarray(ranking.per_layer_scores).astype("<f8").tobytes()]
    return b"".join(parts)


def read_ctkv(data: bytes, chunk_id: str = "chunk"):
    """Parse CTKV bytes -> (KvChunk, ImportanceRanking | None) with the
    reference's validation (ct/cachepool.py:186-230)."""
    if len(data) < HEADER.size:
        raise IoError("truncated CTKV header")
    magic, version, l, n, h, d, dtype, flags = HEADER.unpack_from(data)
    if magic != MAGIC:
        raise IoError(f"bad magic {magic!r}")
    if version != VERSION:
        raise IoError(f"unsupported CTKV version {version}")
    if not flags & FLAG_PRE_ROPE:
        raise IoError("chunk keys are not marked pre-RoPE")
    base = HEADER.size + l * layer_bytes(n, h, d)
    if len(data) not in (base, base + ranking_block_bytes(l, n)):
        raise IoError(f"CTKV length {len(data)} matches neither bare nor ranked layout for "
                      f"geometry L={l} N={n} H={h} D={d}")
    payload = np.frombuffer(data, dtype="<f4", count=l * 2 * n * h * d,
                            offset=HEADER.size).reshape(l, 2, n, h, d)
    chunk = KvChunk(chunk_id, tuple(SeqTensor(payload[i, 0].copy()) for i in range(l)),
                    tuple(SeqTensor(payload[i, 1].copy()) for i in range(l)),
                    dtype_code=DtypeCode(dtype))
    ranking = None
    if len(data) > base:
        (alpha,) = struct.unpack_from("<d", data, base)
        off = base + 8
        orders = np.frombuffer(data, dtype="<u4", count=l * n, offset=off).reshape(l, n)
        off += l * n * 4
        agg = np.frombuffer(data, dtype="<u4", count=n, offset=off)
        off += n * 4
        scores = np.frombuffer(data, dtype="<f8", count=l * n, offset=off).reshape(l, n)
        ranking = ImportanceRanking(per_layer_scores=scores.copy(),
                                    per_layer_order=orders.astype(np.int64),
                                    aggregate_order=agg.astype(np.int64), alpha=alpha,
                                    n_tokens=n)
    return chunk, ranking


def pool_from_ctkv(files, location: str = "pinned", dtype=torch.bfloat16, tokens=None,
                   device="cuda"):
    """Build a KvPool from ranked CTKV files (paths or bytes).  `tokens` gives
    each chunk's source token ids (the format does not carry them,
    ct/kvcore.py:121-123); without them the pool still serves fetches."""
    from .pool import KvPool
    chunks, ranks = [], []
    for i, f in enumerate(files):
        if isinstance(f, (str, Path)):
            try:
                data = Path(f).read_bytes()
            except OSError as e:
                raise IoError(f"cannot read {f}: {e}") from e
            cid = Path(f).stem
        else:
            data, cid = f, f"chunk{i}"
        chunk, rk = read_ctkv(data, cid)
        if rk is None:
            raise InvalidPlan(f"{cid} has no ranking block; analyze it first")
        # without source tokens the chunk stays fetch-only: engines refuse to
        # recompute it (InvalidPlan) instead of recomputing token id 0
        src = None if tokens is None else np.asarray(tokens[i], dtype=np.int64)
        chunk = KvChunk(chunk.chunk_id, chunk.keys_raw, chunk.values, chunk.dtype_code, src)
        chunks.append(DeviceChunk.from_host(chunk, dtype=dtype, device=device))
        ranks.append(rk)
    return KvPool(chunks, ranks, location, device=device)
