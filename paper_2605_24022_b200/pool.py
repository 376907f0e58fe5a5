"""(2) Importance-ordered KV pool and sparse transfer.

The reference stores each chunk token-major in a CTKV file and fetches the
keep set (complement of the recompute set) as coalesced byte ranges --
~400 ranges per (chunk, layer) at config-2 size (ct/cachepool.py:409-481,
SURVEY F8).  Here each chunk's rows are stored in its AGGREGATE IMPORTANCE
ORDER (ct/spectral.py:149-159), K row then V row, layer-major:

    data[c, l, p, 0|1, H, D] = K|V of token aggregate_order[c][p] at layer l

so for any ratio r the keep set of (c, l) is the contiguous tail
p in [ceil(rN), N): ONE copy-engine transfer per (chunk, layer), and the
deferred-RoPE blend kernel reads it with the permutation aggregate_order[k:].
The pool lives in HBM (`location="hbm"`) or pinned host memory
(`location="pinned"`, copied by the copy engines on a side stream).
Byte accounting matches the reference: bytes moved per (chunk, layer) =
|keep| * H * D * dsize * 2 (ct/cachepool.py:434).
"""

from __future__ import annotations

import os
import threading
import time
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _dev, _lib
from .errors import InvalidParam, InvalidPlan, IoError, NotFound
from .spectral import ImportanceRanking, selection_count


@dataclass(frozen=True)
class SparseFetchPlan:
    """Byte-exact plan for one (chunk, layer) at ratio r (ct/cachepool.py:236-255).

    byte_ranges are (offset, length) into the pool's flat byte image; with the
    importance-ordered layout there is exactly one range (or none)."""
    chunk_id: str
    layer: int
    keep_indices: np.ndarray
    byte_ranges: tuple
    expected_bytes: int
    keep_count: int


class KvPool:
    """Importance-ordered pool of equal-geometry chunks."""

    def __init__(self, chunks, rankings, location: str = "hbm", device=None,
                 resident_layers: int = 0):
        """resident_layers (pinned pools): the first n layers' importance-
        ordered rows are also kept in HBM, so a request's earliest layers --
        whose transfer nothing can overlap -- read them in place (tiered
        placement; the other layers stream over PCIe)."""
        if len(chunks) == 0 or len(chunks) != len(rankings):
            raise InvalidPlan("need one ranking per chunk")
        if location not in ("hbm", "pinned"):
            raise InvalidParam(f"unknown pool location {location!r}")
        device = device or _dev.require_cuda()
        c0 = chunks[0]
        L, N, H, D = c0.keys.shape
        for c, rk in zip(chunks, rankings):
            if tuple(c.keys.shape) != (L, N, H, D):
                raise InvalidParam("pool chunks must share one geometry")
            if rk.n_tokens != N:
                raise InvalidPlan("ranking/chunk token counts disagree")
        self.location = location
        self.device = torch.device(device)
        if self.device.type == "cuda" and self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        self.dtype = c0.keys.dtype
        self.C, self.L, self.N, self.H, self.D = len(chunks), L, N, H, D
        self.chunk_ids = [c.chunk_id for c in chunks]
        self.rankings = list(rankings)
        self.esize = torch.empty((), dtype=self.dtype).element_size()
        self.row_bytes = H * D * self.esize
        self.agg = torch.stack([rk.aggregate_device(self.device) for rk in rankings]).contiguous()
        # source token ids per chunk; a chunk restored from a CTKV file without
        # them (the format does not carry tokens, ct/kvcore.py:121-123) serves
        # sparse fetches but cannot be recomputed (engines raise InvalidPlan,
        # ct/toymodel.py:243-244)
        self.has_tokens = [c.tokens is not None or c.source_tokens is not None for c in chunks]

        def dev_tokens(c):
            if c.tokens is not None:
                return c.tokens
            if c.source_tokens is not None:
                return torch.as_tensor(np.asarray(c.source_tokens, np.int32), device=self.device)
            return torch.zeros(N, dtype=torch.int32, device=self.device)  # never read
        self.tokens = torch.stack([dev_tokens(c) for c in chunks]).contiguous()
        self.tokens_host = np.stack([np.asarray(c.source_tokens, np.int64)
                                     if c.source_tokens is not None else np.zeros(N, np.int64)
                                     for c in chunks])
        shape = (self.C, L, N, 2, H, D)
        dev_img = torch.empty(shape, dtype=self.dtype, device=self.device)
        self._permute(chunks, dev_img)
        self.resident_layers = 0 if location == "hbm" else max(0, min(int(resident_layers), L))
        self.resident = None
        if location == "hbm":
            self.data = dev_img
        else:
            self.data = torch.empty(shape, dtype=self.dtype, pin_memory=True)
            self.data.copy_(dev_img)
            if self.resident_layers:
                self.resident = dev_img[:, :self.resident_layers].clone()
            del dev_img
        self._stats_lock = threading.Lock()
        self.io_stats = {"bytes_read": 0, "reads": 0}

    def _permute(self, chunks, dev_img) -> None:
        """Offline: rows into importance order with ct_pool_permute -- one
        launch for all chunks when they are slices of one [C, L, N, H, D]
        batch (the offline stage's layout), else one launch per chunk."""
        L, N = self.L, self.N
        ks, vs = [c.keys for c in chunks], [c.values for c in chunks]
        for t in ks + vs:
            if t.device != self.device or not t.is_contiguous() or t.dtype != self.dtype:
                raise InvalidParam("pool chunks must be contiguous tensors of one dtype on the "
                                   "pool's device")
        row = self.row_bytes
        st = _dev.stream_handle()

        def uniform(ts):
            if len(ts) < 2:
                return 0
            d = ts[1].data_ptr() - ts[0].data_ptr()
            ok = d > 0 and all(b.data_ptr() - a.data_ptr() == d for a, b in zip(ts, ts[1:]))
            return d if ok else 0
        dk, dv = uniform(ks), uniform(vs)
        # chunk c's rows live at base + c * ld_chunk exactly when the spacing
        # of the chunks' own data pointers is uniform (checked above)
        groups = ([(0, self.C, dk)] if dk and dk == dv
                  else [(ci, 1, L * N * row) for ci in range(self.C)])
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for c0, nc, ld_chunk in groups:
            _lib.call("ct_pool_permute", _dev.ptr(ks[c0]), _dev.ptr(vs[c0]), nc, L, N, row,
                      N * row, ld_chunk, row, _dev.ptr(self.agg[c0]), _dev.ptr(dev_img[c0]), st)
        ev[1].record()
        self.permute_launches = len(groups)
        self._permute_events = ev

    @property
    def permute_ms(self) -> float:
        """Device time of the offline permute launches (synchronises)."""
        ev = self._permute_events
        ev[1].synchronize()
        return ev[0].elapsed_time(ev[1])

    # -- geometry ----------------------------------------------------------
    @property
    def nbytes(self) -> int:
        return self.data.numel() * self.esize

    def chunk_index(self, chunk_id) -> int:
        if isinstance(chunk_id, int):
            return chunk_id
        try:
            return self.chunk_ids.index(chunk_id)
        except ValueError:
            raise NotFound(f"chunk {chunk_id!r} not in pool") from None

    def offset_bytes(self, c: int, l: int, p: int) -> int:
        return (((c * self.L + l) * self.N + p) * 2) * self.row_bytes

    def tail_ptr(self, c: int, l: int, k: int) -> int:
        return self.data.data_ptr() + self.offset_bytes(c, l, k)

    def resident_tail_ptr(self, c: int, l: int, k: int) -> int:
        """HBM address of a resident layer's keep tail (l < resident_layers)."""
        if not 0 <= l < self.resident_layers:
            raise InvalidParam(f"layer {l} is not HBM-resident")
        R = self.resident_layers
        return self.resident.data_ptr() + (((c * R + l) * self.N + k) * 2) * self.row_bytes

    # -- reference-shaped sparse API (ct/cachepool.py:409-481) ------------------
    def plan_sparse_fetch(self, chunk_id, layer: int, r: float) -> SparseFetchPlan:
        c = self.chunk_index(chunk_id)
        if not 0 <= layer < self.L:
            raise InvalidParam(f"layer {layer} out of range [0, {self.L})")
        k = selection_count(r, self.N)
        keep = np.sort(self.rankings[c].aggregate_order[k:])
        n_keep = self.N - k
        length = n_keep * 2 * self.row_bytes
        ranges = ((self.offset_bytes(c, layer, k), length),) if n_keep else ()
        return SparseFetchPlan(self.chunk_ids[c], layer, keep, ranges, n_keep * self.row_bytes * 2,
                               n_keep)

    # -- tier model / profiling (ct/cachepool.py:483-529) -----------------------
    def modeled_fetch_time(self, plan: SparseFetchPlan, tier=None) -> float:
        """Modelled read time of a plan on `tier` (default: the cpu-mem preset
        for a pinned pool, gpu-sim for an HBM pool)."""
        from .pipesim import TIER_PRESETS
        tier = tier or TIER_PRESETS["cpu-mem" if self.location == "pinned" else "gpu-sim"]
        return tier.read_time(plan.expected_bytes)

    def measure_transfer_cost(self, tier, sample_bytes: int,
                              bytes_per_token: int | None = None) -> float:
        """t_i for `tier` exactly as the reference computes it (scheduler.calibrate
        calls this when no profile is injected); bytes_per_token defaults to
        the reference's f32 K+V CTKV row.  The B200 PCIe rate itself is
        measured by scheduler.measure_h2d_per_token."""
        if bytes_per_token is None:
            # the reference's CTKV row (f32 K + V, ct/cachepool.py:146-152,505),
            # as cachepool.token_row_bytes and pipesim.layer_keep_bytes charge
            # it -- not this pool's storage width
            bytes_per_token = self.H * self.D * 4 * 2
        return transfer_cost_per_token(tier, sample_bytes, bytes_per_token)

    def fetch_sparse(self, plan: SparseFetchPlan, stream=None):
        """Move exactly the planned bytes to HBM; return (K [keep,H,D], V, keep)
        in ascending token order like the reference."""
        c = self.chunk_index(plan.chunk_id)
        if plan.expected_bytes != len(plan.keep_indices) * self.row_bytes * 2:
            raise InvalidPlan("expected_bytes disagrees with keep_indices")
        n_keep = plan.keep_count
        if n_keep == 0:
            return None, None, plan.keep_indices
        k = self.N - n_keep
        src = self.tail_ptr(c, plan.layer, k)
        nbytes = plan.byte_ranges[0][1]
        # every allocation, copy and gather on ONE stream (the caller's, default
        # current): the staging buffer's memory cannot be reused by another
        # stream's allocation while the copy / gather still read it
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.stream(st):
            stage = torch.empty((n_keep, 2, self.H, self.D), dtype=self.dtype, device=self.device)
            if self.location == "pinned":
                _lib.call("ct_copy_ranges_h2d", ctypes_ptr_array([stage.data_ptr()]),
                          ctypes_ptr_array([src]), ctypes_i64_array([nbytes]), 1,
                          _dev.stream_handle(st))
            else:
                off = self.offset_bytes(c, plan.layer, k) // self.esize
                stage.view(-1).view(torch.uint8).copy_(
                    self.data.view(-1)[off: off + nbytes // self.esize].view(torch.uint8))
            # un-permute: output row i = token keep[i] = tail row rank[keep[i]] - k
            rank = np.argsort(self.rankings[c].aggregate_order)
            rows = torch.as_tensor((rank[plan.keep_indices] - k).astype(np.int32),
                                   device=self.device)
            kv = torch.empty_like(stage)
            _lib.call("ct_gather_rows", _dev.ptr(stage), _dev.ptr(rows), n_keep,
                      2 * self.row_bytes, _dev.ptr(kv), _dev.stream_handle(st))
        with self._stats_lock:
            self.io_stats["bytes_read"] += nbytes
            self.io_stats["reads"] += 1
        return kv[:, 0], kv[:, 1], plan.keep_indices


def transfer_cost_per_token(tier, sample_bytes: int, bytes_per_token: int) -> float:
    """Per-token transfer cost t_i of a tier (ct/cachepool.py:489-529): the
    analytic model for simulated tiers, a timed sequential read of
    sample_bytes for file-backed ones (tier.backing = directory)."""
    if sample_bytes <= 0:
        raise InvalidParam("sample_bytes must be > 0")
    tokens = sample_bytes / bytes_per_token
    if tier.backing is None:
        return tier.read_time(sample_bytes) / tokens
    try:
        root = Path(tier.backing)
        root.mkdir(parents=True, exist_ok=True)
        probe = root / ".transfer_probe"
        payload = os.urandom(min(sample_bytes, 1 << 20))
        with open(probe, "wb") as f:
            written = 0
            while written < sample_bytes:
                piece = payload[: sample_bytes - written]
                f.write(piece)
                written += len(piece)
            f.flush()
            os.fsync(f.fileno())
        start = time.perf_counter()
        with open(probe, "rb") as f:
            while f.read(1 << 20):
                pass
        elapsed = time.perf_counter() - start
        probe.unlink(missing_ok=True)
    except OSError as e:
        raise IoError(f"transfer probe failed on {tier.backing}: {e}") from e
    return max(elapsed, 1e-12) / tokens


def ctypes_ptr_array(vals):
    import ctypes
    return (ctypes.c_void_p * len(vals))(*vals)


def ctypes_i64_array(vals):
    import ctypes
    return (ctypes.c_int64 * len(vals))(*vals)
