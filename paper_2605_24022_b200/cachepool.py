"""Reference-shaped chunk registry (`CachePool`, ct/cachepool.py:283-529) over
the B200 path.

The reference keeps every chunk as a CTKV file image (in memory or on a
file-backed tier), plans a layer's reused rows as coalesced byte ranges of
that image and reads them back into numpy.  This class keeps the same
registry semantics -- `put_chunk` / `attach_chunk_file` / `get_ranking` /
`get_full` / `plan_sparse_fetch` / `fetch_sparse` / `modeled_*` /
`measure_transfer_cost`, `io_stats` with exact byte accounting, per-chunk-id
writer locks, `AlreadyExists` / `NotFound` / `IoError` -- with two B200
differences:

* `fetch_sparse` stages exactly the planned byte ranges into pinned host
  memory (direct `preadv` from a file-backed tier, no intermediate join) and
  moves them to HBM with ONE copy-engine transfer; it returns device
  tensors K, V `[keep, H, D]` f32 in ascending token order (bit-identical
  to the reference's rows) and the keep indices.
* `to_kv_pool(location, dtype)` converts the registry into the
  importance-ordered `KvPool` the online engine uses (one contiguous tail
  per (chunk, layer) instead of ~400 ranges).

Planning (`plan_sparse_fetch`) is integer work on the host, vectorised with
numpy (the reference loops over tokens in Python, 1.58 ms per chunk-layer at
config 2).
"""

from __future__ import annotations

import os
import threading
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _dev, _lib
from .ctkv import HEADER, layer_bytes, read_ctkv, write_ctkv
from .errors import AlreadyExists, InvalidParam, InvalidPlan, IoError, NotFound, ShapeError
from .pool import SparseFetchPlan, ctypes_i64_array, ctypes_ptr_array, transfer_cost_per_token
from .spectral import selection_count

ROW_DTYPE_SIZE = 4  # CTKV payload is f32 (ct/cachepool.py:146-152)


def token_row_bytes(h: int, d: int) -> int:
    return h * d * ROW_DTYPE_SIZE


@dataclass
class _Stored:
    tier: object
    geometry: tuple          # (L, N, H, D)
    path: Path | None        # file-backed tier
    blob: bytes | None       # in-memory tier
    ranking: object
    file_bytes: int
    modeled_write_s: float
    source_tokens: np.ndarray | None = None


def _ranges(keep: np.ndarray, k_base: int, v_base: int, row: int) -> tuple:
    """Coalesced (offset, length) ranges of the keep rows in the K block then
    the V block, a K tail abutting the V head merged (ct/cachepool.py:258-266,
    416-429), vectorised."""
    if keep.size == 0:
        return ()
    brk = np.flatnonzero(np.diff(keep) != 1) + 1
    starts = keep[np.concatenate([[0], brk])]
    counts = np.diff(np.concatenate([[0], brk, [keep.size]]))
    out = []
    for base in (k_base, v_base):
        for s, c in zip((base + starts * row).tolist(), (counts * row).tolist()):
            if out and s == out[-1][0] + out[-1][1]:
                out[-1] = (out[-1][0], out[-1][1] + c)
            else:
                out.append((s, c))
    return tuple(out)


class CachePool:
    """Chunk registry across tiers with byte-accounted sparse fetches into HBM.
    Concurrent readers are safe; writes take the registry lock plus a per
    chunk-id lock (ct/cachepool.py:283-304)."""

    def __init__(self, device=None):
        self._chunks: dict[str, _Stored] = {}
        self._registry_lock = threading.Lock()
        self._id_locks: dict[str, threading.Lock] = {}
        self._stats_lock = threading.Lock()
        self.io_stats = {"bytes_read": 0, "reads": 0, "bytes_written": 0, "writes": 0}
        self._device = device

    def _count_io(self, key: str, n_bytes: int) -> None:
        with self._stats_lock:
            self.io_stats[f"bytes_{key}"] += n_bytes
            self.io_stats["reads" if key == "read" else "writes"] += 1

    # -- write path (ct/cachepool.py:306-374) ----------------------------------
    def put_chunk(self, chunk, ranking, tier) -> str:
        """Serialise a chunk (with its ranking) into the given tier."""
        if ranking.n_tokens != chunk.token_count or ranking.n_layers != chunk.n_layers:
            raise ShapeError("chunk and ranking disagree on N or L")
        cid = chunk.chunk_id
        with self._registry_lock:
            lock = self._id_locks.setdefault(cid, threading.Lock())
        with lock:
            if cid in self._chunks:
                raise AlreadyExists(f"chunk {cid!r} already stored")
            data = write_ctkv(chunk, ranking)
            path = blob = None
            if tier.backing is not None:
                try:
                    root = Path(tier.backing)
                    root.mkdir(parents=True, exist_ok=True)
                    path = root / f"{cid}.ctkv"
                    path.write_bytes(data)
                except OSError as e:
                    raise IoError(f"failed to write chunk {cid!r}: {e}") from e
            else:
                blob = data
            stored = _Stored(tier, (chunk.n_layers, chunk.token_count, chunk.n_heads,
                                    chunk.head_dim), path, blob, ranking, len(data),
                             tier.write_time(len(data)),
                             getattr(chunk, "source_tokens", None))
            with self._registry_lock:
                self._chunks[cid] = stored
            self._count_io("written", len(data))
        return cid

    def attach_chunk_file(self, path, tier) -> str:
        """Register an existing ranked CTKV file under its stem id."""
        path = Path(path)
        cid = path.stem
        try:
            data = path.read_bytes()
        except OSError as e:
            raise IoError(f"cannot read {path}: {e}") from e
        chunk, ranking = read_ctkv(data, chunk_id=cid)
        if ranking is None:
            raise InvalidPlan(f"{path} has no ranking block; analyze it first")
        with self._registry_lock:
            if cid in self._chunks:
                raise AlreadyExists(f"chunk {cid!r} already stored")
            self._chunks[cid] = _Stored(
                tier, (chunk.n_layers, chunk.token_count, chunk.n_heads, chunk.head_dim),
                path if tier.backing is not None else None,
                None if tier.backing is not None else data, ranking, len(data),
                tier.write_time(len(data)))
        return cid

    # -- lookups (ct/cachepool.py:376-407) -------------------------------------
    def _stored(self, chunk_id: str) -> _Stored:
        try:
            return self._chunks[chunk_id]
        except KeyError:
            raise NotFound(f"chunk {chunk_id!r} not in pool") from None

    def chunk_ids(self) -> list[str]:
        return sorted(self._chunks)

    def geometry(self, chunk_id: str) -> tuple:
        return self._stored(chunk_id).geometry

    def file_bytes(self, chunk_id: str) -> int:
        return self._stored(chunk_id).file_bytes

    def modeled_write_time(self, chunk_id: str) -> float:
        return self._stored(chunk_id).modeled_write_s

    def get_ranking(self, chunk_id: str):
        return self._stored(chunk_id).ranking

    def _raw(self, stored: _Stored) -> bytes:
        if stored.blob is not None:
            return stored.blob
        try:
            return stored.path.read_bytes()
        except OSError as e:
            raise IoError(f"failed to read {stored.path}: {e}") from e

    def get_full(self, chunk_id: str):
        """Deserialise the whole chunk, bit-exact (host KvChunk)."""
        stored = self._stored(chunk_id)
        data = self._raw(stored)
        self._count_io("read", len(data))
        chunk, _ = read_ctkv(data, chunk_id=chunk_id)
        return chunk

    # -- sparse path (ct/cachepool.py:409-487) ---------------------------------
    def plan_sparse_fetch(self, chunk_id: str, layer: int, r: float) -> SparseFetchPlan:
        """The layer's reused-KV byte ranges of the CTKV image at ratio r."""
        stored = self._stored(chunk_id)
        l, n, h, d = stored.geometry
        if not 0 <= layer < l:
            raise InvalidParam(f"layer {layer} out of range [0, {l})")
        k = selection_count(r, n)
        keep = np.sort(np.asarray(stored.ranking.aggregate_order, np.int64)[k:])
        row = token_row_bytes(h, d)
        k_base = HEADER.size + layer * layer_bytes(n, h, d)
        ranges = _ranges(keep, k_base, k_base + n * row, row)
        return SparseFetchPlan(chunk_id, layer, keep, ranges, int(keep.size) * row * 2,
                               int(keep.size))

    def fetch_sparse(self, plan: SparseFetchPlan, stream=None):
        """Read exactly the planned ranges into pinned memory, one H2D copy,
        -> (K [keep,H,D] f32 device, V, keep_indices); None tensors for an
        empty plan.  Bytes read always equal plan.expected_bytes."""
        stored = self._stored(plan.chunk_id)
        l, n, h, d = stored.geometry
        keep = np.asarray(plan.keep_indices, np.int64)
        row = token_row_bytes(h, d)
        if plan.expected_bytes != keep.size * row * 2:
            raise InvalidPlan("expected_bytes disagrees with keep_indices")
        if keep.size == 0:
            return None, None, keep
        if sum(length for _, length in plan.byte_ranges) != plan.expected_bytes:
            raise InvalidPlan("byte ranges disagree with expected_bytes")
        stage = torch.empty(plan.expected_bytes, dtype=torch.uint8, pin_memory=True)
        view = stage.numpy()
        pos = 0
        if stored.path is not None:
            try:
                fd = os.open(stored.path, os.O_RDONLY)
                try:
                    for off, length in plan.byte_ranges:
                        got = os.preadv(fd, [memoryview(view[pos:pos + length])], off)
                        if got != length:
                            raise IoError(f"short read at {off} in {stored.path}")
                        pos += length
                finally:
                    os.close(fd)
            except OSError as e:
                raise IoError(f"failed sparse read of {stored.path}: {e}") from e
        else:
            blob = np.frombuffer(stored.blob, dtype=np.uint8)
            for off, length in plan.byte_ranges:
                if off + length > blob.size:
                    raise InvalidPlan("byte range beyond stored chunk")
                view[pos:pos + length] = blob[off:off + length]
                pos += length
        self._count_io("read", pos)
        dev = torch.device(self._device) if self._device is not None else _dev.require_cuda()
        out = torch.empty(plan.expected_bytes, dtype=torch.uint8, device=dev)
        _lib.call("ct_copy_ranges_h2d", ctypes_ptr_array([out.data_ptr()]),
                  ctypes_ptr_array([stage.data_ptr()]), ctypes_i64_array([pos]), 1,
                  _dev.stream_handle(stream))
        # the staging buffer must outlive the async copy
        (stream or torch.cuda.current_stream(dev)).synchronize()
        kv = out.view(torch.float32).view(2, keep.size, h, d)
        return kv[0], kv[1], keep

    def modeled_fetch_time(self, plan: SparseFetchPlan) -> float:
        return self._stored(plan.chunk_id).tier.read_time(plan.expected_bytes)

    # -- profiling (ct/cachepool.py:489-529) ------------------------------------
    def measure_transfer_cost(self, tier, sample_bytes: int,
                              bytes_per_token: int | None = None) -> float:
        if sample_bytes <= 0:
            raise InvalidParam("sample_bytes must be > 0")
        if bytes_per_token is None:
            ids = self.chunk_ids()
            if not ids:
                raise InvalidParam("pool empty: pass bytes_per_token explicitly")
            _, _, h, d = self.geometry(ids[0])
            bytes_per_token = token_row_bytes(h, d) * 2
        return transfer_cost_per_token(tier, sample_bytes, bytes_per_token)

    # -- the online engine's layout ----------------------------------------------
    def to_kv_pool(self, chunk_ids=None, location: str = "hbm", dtype=torch.bfloat16,
                   tokens=None):
        """Importance-ordered KvPool of the given (default: all) chunks for
        pipeline.SelectivePrefillEngine.  `tokens[i]` = source token ids when
        the chunk was stored without them."""
        from .kvcore import DeviceChunk, KvChunk
        from .pool import KvPool
        ids = list(chunk_ids) if chunk_ids is not None else self.chunk_ids()
        dev = torch.device(self._device) if self._device is not None else _dev.require_cuda()
        chunks, ranks = [], []
        for i, cid in enumerate(ids):
            stored = self._stored(cid)
            host = self.get_full(cid)
            src = tokens[i] if tokens is not None else stored.source_tokens
            src = None if src is None else np.asarray(src)  # None: fetch-only chunk
            host = KvChunk(cid, host.keys_raw, host.values, host.dtype_code, src)
            chunks.append(DeviceChunk.from_host(host, dtype=dtype, device=dev))
            ranks.append(stored.ranking)
        return KvPool(chunks, ranks, location, device=dev)
