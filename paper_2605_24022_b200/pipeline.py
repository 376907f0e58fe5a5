"""Serving-shaped engines for repeated requests over a resident chunk pool.

`SelectivePrefillEngine` is the online path of ct/toymodel.py:223-311 with
every buffer preallocated, the selection plan, the sparse transfer and the
deferred-RoPE blend wired to a `KvPool`:

  * pool in HBM ("hbm"): K3 reads each (chunk, layer) keep tail in place.
  * pool in pinned host memory ("pinned"): all (chunk, layer) tails are issued
    up front as ONE cudaMemcpyAsync each on a copy stream (copy engines, no SM
    time); layer l's blend waits only on layer l's copy event, so PCIe runs
    flat out underneath the per-layer recompute (the three-stream overlap of
    ct/pipesim.py:196-241, collection layer = layer 0's transfer).

`FullPrefillEngine` is the full-recompute baseline built from the same
kernels (every token a query, dense causal).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _dev, _lib
from .errors import InvalidPlan
from .model import GpuModel
from .pool import KvPool
from .prefill import NORM_EPS, LayerBuffers, run_layers  # noqa: F401
from .rope import rope_table
from .spectral import selection_count


class KernelTimer:
    """CUDA-event pairs around named launches on the current stream."""

    def __init__(self):
        self.enabled = False
        self.events: dict = {}

    def start(self, name):
        if not self.enabled:
            return None
        s = torch.cuda.Event(enable_timing=True)
        s.record()
        return s

    def stop(self, name, s):
        if s is None:
            return
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.events.setdefault(name, []).append((s, e))

    def mean_ms(self, name) -> float:
        ev = self.events.get(name, [])
        if not ev:
            return float("nan")
        return float(np.mean([s.elapsed_time(e) for s, e in ev]))

    def count(self, name) -> int:
        return len(self.events.get(name, []))

    def reset(self):
        self.events = {}


class SelectivePrefillEngine:
    """One request at a time: the context is `n_chunks` chunks of the pool (by
    default all of them, in pool order) + a suffix of `suffix_len` tokens.
    With a corpus pool (more chunks than a request uses) `bind(chunk_ids)`
    points the engine at the request's chunks -- RAG requests drawing
    different documents from one shared, importance-ordered KV corpus -- and
    reuses every device buffer."""

    def __init__(self, model: GpuModel, pool: KvPool, r: float, suffix_len: int,
                 timer: KernelTimer | None = None, n_chunks: int | None = None,
                 ring_layers: int = 4):
        cfg = model.config
        if (pool.L, pool.H, pool.D) != (cfg.n_layers, cfg.kv_heads, cfg.head_dim):
            raise ValueError("pool geometry disagrees with model")
        self.model, self.pool, self.r, self.S = model, pool, r, suffix_len
        self.timer = timer or KernelTimer()
        dev = model.device
        C = pool.C if n_chunks is None else int(n_chunks)
        if not 1 <= C <= pool.C:
            raise ValueError(f"a request uses 1..{pool.C} chunks of this pool, not {C}")
        N, L, H, D = pool.N, pool.L, pool.H, pool.D
        self.C = C
        self.k = selection_count(r, N)
        self.n_keep = N - self.k
        self.history = C * N
        self.n_ctx = self.history + suffix_len
        self.n_rec = C * self.k
        self.A = self.n_rec + suffix_len
        dt = model.dtype
        self.cache = torch.empty((L, 2, self.n_ctx, H, D), dtype=dt, device=dev)
        self.caches = [(self.cache[l, 0], self.cache[l, 1]) for l in range(L)]
        self.buffers = LayerBuffers(model, self.A, dev)
        self.positions = torch.empty(self.A, dtype=torch.int32, device=dev)
        self.tokens = torch.zeros(self.A, dtype=torch.int32, device=dev)  # suffix defaults to id 0
        self.positions[self.n_rec:] = torch.arange(self.history, self.n_ctx, dtype=torch.int32,
                                                   device=dev)
        self.keep = torch.empty(C * self.n_keep, dtype=torch.int32, device=dev)
        self.keep_src = torch.empty_like(self.keep)
        offsets = np.arange(C + 1, dtype=np.int64) * N
        meta = np.concatenate([offsets, np.full(C, self.k), np.arange(C + 1) * self.k,
                               np.arange(C + 1) * self.n_keep]).astype(np.int64)
        self.meta = torch.as_tensor(meta, device=dev)
        self.table = rope_table(cfg.rope_params, self.n_ctx, "f64" if dt == torch.float32
                                else "f32", dev)
        self.pinned = pool.location == "pinned"
        self.row_elems = H * D
        # pinned pool: layers >= res stream over PCIe through a ring of
        # `ring` staging slots (a layer's copy may start once the blend of
        # the layer that last used its slot has run); layers < res are the
        # pool's HBM-resident tier
        self.res = pool.resident_layers if self.pinned else 0
        self.ring = max(1, min(int(ring_layers), L - self.res)) if self.pinned else 0
        if self.pinned:
            self.stage = torch.empty((self.ring, C, max(self.n_keep, 1), 2, H, D), dtype=dt,
                                     device=dev)
            self.copy_stream = torch.cuda.Stream(device=dev)
            self.copy_done = [torch.cuda.Event() for _ in range(L)]
            self.slot_free = [torch.cuda.Event() for _ in range(L)]
            self.step_start = torch.cuda.Event()
            self.h2d_bytes = (L - self.res) * C * self.n_keep * 2 * pool.row_bytes
        else:
            self.h2d_bytes = 0
        self.n_segs = C if self.n_keep else 0
        self.launches_per_step = None
        self.record_timeline = False
        self._events: dict = {}
        self.graph = None
        # the request's chunks: aggregate orders and token ids gathered from
        # the pool (device), transfer / blend parameters built on the host
        self.agg = torch.empty((C, N), dtype=torch.int32, device=dev)
        self.chunk_tokens = torch.empty((C, N), dtype=torch.int32, device=dev)
        self.chunk_ids = None
        self.bind(list(range(C)))

    def bind(self, chunk_ids) -> None:
        """Point the engine at pool chunks `chunk_ids` (len == n_chunks, pool
        indices or ids), in context order.  Asynchronous on the current stream;
        not allowed while a captured graph is in use (its parameters are baked)."""
        pool, C, N = self.pool, self.C, self.pool.N
        idx = [pool.chunk_index(c) for c in chunk_ids]
        if len(idx) != C:
            raise ValueError(f"request needs exactly {C} chunks, got {len(idx)}")
        for ci in idx:  # ct/toymodel.py:243-244
            if self.k and not pool.has_tokens[ci]:
                raise InvalidPlan(f"chunk {pool.chunk_ids[ci]!r} lacks source_tokens; "
                                  "cannot recompute")
        if self.graph is not None and idx != self.chunk_ids:
            raise RuntimeError("bind() would change a captured graph's parameters")
        self.chunk_ids = idx
        # pinned + non_blocking: binding the next request never waits for the
        # GPU to drain the current one
        sel = torch.tensor(idx, dtype=torch.long).pin_memory().to(self.agg.device,
                                                                  non_blocking=True)
        torch.index_select(pool.agg, 0, sel, out=self.agg)
        torch.index_select(pool.tokens, 0, sel, out=self.chunk_tokens)
        L, H, D, esz = pool.L, pool.H, pool.D, pool.esize
        if self.pinned:
            nbytes = self.n_keep * 2 * pool.row_bytes
            self.copy_args = [None] * L
            for l in range(self.res, L):
                dst = [self.stage[self._slot(l), c].data_ptr() for c in range(C)]
                src = [pool.tail_ptr(ci, l, self.k) for ci in idx]
                self.copy_args[l] = ((ctypes.c_void_p * C)(*dst), (ctypes.c_void_p * C)(*src),
                                     (ctypes.c_int64 * C)(*([nbytes] * C)))
        # per-layer K3 segments (kernel parameters), in launches of at most
        # CT_MAX_SEGMENTS segments each
        self.segs = []
        for l in range(L):
            segs = []
            for c, ci in enumerate(idx):
                if self.n_keep == 0:
                    continue
                if not self.pinned:
                    base = pool.tail_ptr(ci, l, self.k)
                elif l < self.res:
                    base = pool.resident_tail_ptr(ci, l, self.k)
                else:
                    base = self.stage[self._slot(l), c].data_ptr()
                tok = self.agg.data_ptr() + (c * N + self.k) * 4
                segs.append(_lib.Segment(base, base + H * D * esz, tok, self.n_keep, c * N, 0))
            groups = [segs[i:i + _lib.CT_MAX_SEGMENTS]
                      for i in range(0, len(segs), _lib.CT_MAX_SEGMENTS)]
            self.segs.append([((_lib.Segment * len(g))(*g), len(g)) for g in groups])

    # real three-stream timeline (ct/pipesim.py Timeline schema) ------------------
    def _ev(self, stream: str, layer: int, edge: int) -> torch.cuda.Event:
        key = (stream, layer, edge)
        ev = self._events.get(key)
        if ev is None:
            ev = torch.cuda.Event(enable_timing=True)
            self._events[key] = ev
        return ev

    def _hook(self, l: int, phase: str) -> None:
        # recompute l = QKV projection + RoPE/scatter of the selected rows;
        # forward l = blend (waits on transfer l) + attention + projections/MLP
        if phase == "start":
            self._ev("recompute", l, 0).record()
        elif phase == "recomputed":
            self._ev("recompute", l, 1).record()
            if not self.pinned or self.n_segs == 0:
                self._ev("forward", l, 0).record()
        else:
            self._ev("forward", l, 1).record()

    def _step_hook(self, user):
        if not self.record_timeline:
            return user
        if user is None:
            return self._hook

        def both(l, phase):
            self._hook(l, phase)
            user(l, phase)
        return both

    def timeline(self):
        """Timeline of the last step recorded with record_timeline=True, in
        seconds from the step start (ct/pipesim.py:93-105 schema); audit it
        with pipesim.validate_timeline."""
        from .pipesim import Timeline, TimelineEvent
        t0 = self._ev("step", 0, 0)
        events = []
        for l in range(self.pool.L):
            for stream, label in (("transfer", "gather" if l == 0 else "prefetch"),
                                  ("recompute", "recompute+rope"),
                                  ("forward", "fuse")):
                if (stream, l, 0) not in self._events:
                    continue
                s = t0.elapsed_time(self._ev(stream, l, 0)) * 1e-3
                e = t0.elapsed_time(self._ev(stream, l, 1)) * 1e-3
                events.append(TimelineEvent(stream, l, s, e, label))
        return Timeline(tuple(events), max(e.end_s for e in events))

    # algorithmic work per request -------------------------------------------------
    def attention_flops_per_layer(self) -> float:
        pos = self.positions.double().cpu().numpy()
        cfg = self.model.config
        return float(4.0 * cfg.n_heads * cfg.head_dim * np.sum(pos + 1.0))

    def blend_bytes_per_layer(self) -> int:
        # read keep rows (K and V) + write them into the cache
        return 2 * 2 * self.C * self.n_keep * self.pool.row_bytes

    def _slot(self, l: int) -> int:
        return (l - self.res) % self.ring

    def _issue_copy(self, l: int, after=None) -> None:
        """Queue layer l's keep-tail copies (one cudaMemcpyAsync per chunk) on
        the copy stream, after event `after` (the blend that freed its slot)."""
        with torch.cuda.stream(self.copy_stream):
            if after is not None:
                self.copy_stream.wait_event(after)
            if self.record_timeline:
                self._ev("transfer", l, 0).record(self.copy_stream)
            d, s, b = self.copy_args[l]
            _lib.call("ct_copy_ranges_h2d", d, s, b, self.C, _dev.stream_handle(self.copy_stream))
            self.copy_done[l].record(self.copy_stream)
            if self.record_timeline:
                self._ev("transfer", l, 1).record(self.copy_stream)

    def time_transfer(self) -> float:
        """ms of copy-engine time for one request's streamed keep tails alone
        (every streamed layer back to back on the copy stream, no compute);
        h2d_bytes / this = the achieved sparse-transfer rate."""
        if not self.pinned or self.n_segs == 0 or self.res >= self.pool.L:
            return 0.0
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        self.copy_stream.wait_stream(torch.cuda.current_stream())
        s.record(self.copy_stream)
        for l in range(self.res, self.pool.L):
            d, src, b = self.copy_args[l]
            _lib.call("ct_copy_ranges_h2d", d, src, b, self.C,
                      _dev.stream_handle(self.copy_stream))
        e.record(self.copy_stream)
        e.synchronize()
        return s.elapsed_time(e)

    def _reuse(self, l: int) -> None:
        if self.n_segs == 0:
            return
        st = _dev.stream_handle()
        streamed = self.pinned and l >= self.res
        if streamed:
            torch.cuda.current_stream().wait_event(self.copy_done[l])
        if self.pinned and self.record_timeline:
            self._ev("forward", l, 0).record()   # fusion starts once transfer l landed
        t = self.timer.start("blend")
        pool = self.pool
        for arr, n in self.segs[l]:
            _lib.call("ct_gather_rope_blend", arr, n, 2 * self.row_elems,
                      pool.H, pool.D, _dev.ct_dtype(pool.dtype),
                      self.model.config.rope_params.pairing_code, _dev.ptr(self.table),
                      _dev.ptr(self.cache[l, 0]), _dev.ptr(self.cache[l, 1]), self.row_elems, st)
        self.timer.stop("blend", t)
        if streamed and l + self.ring < self.pool.L:
            # slot of layer l is free once this blend ran: refill it with l + ring
            self.slot_free[l].record()
            self._issue_copy(l + self.ring, after=self.slot_free[l])

    def step(self, suffix=None, logits_out: torch.Tensor | None = None,
             hook=None) -> torch.Tensor:
        """One request: suffix (host pinned or device int32 [S]) -> last-row logits.
        hook(layer, phase) (phases "start", "recomputed", "end") runs on the
        host between a layer's launches, e.g. to snapshot `self.buffers`."""
        pool, st = self.pool, _dev.stream_handle()
        C, N = self.C, pool.N
        if self.record_timeline:
            self._ev("step", 0, 0).record()
        if self.pinned and self.n_segs and self.res < pool.L:
            # the first `ring` streamed layers go out before anything else of
            # the request (selection, embedding); the previous request's
            # blends (which read the same slots) precede step_start
            self.step_start.record()
            for i, l in enumerate(range(self.res, min(pool.L, self.res + self.ring))):
                self._issue_copy(l, after=self.step_start if i == 0 else None)
        if suffix is not None and self.S:
            self.tokens[self.n_rec:].copy_(suffix, non_blocking=True)
        m = self.meta
        _lib.call("ct_selection_plan", _dev.ptr(self.agg), _dev.ptr(m[:C + 1]),
                  _dev.ptr(m[C + 1:2 * C + 1]), _dev.ptr(m[2 * C + 1:3 * C + 2]),
                  _dev.ptr(m[3 * C + 2:]), C, N, _dev.ptr(self.positions), _dev.ptr(self.keep),
                  _dev.ptr(self.keep_src), st)
        if self.n_rec:
            _lib.call("ct_gather_rows", _dev.ptr(self.chunk_tokens), _dev.ptr(self.positions),
                      self.n_rec, 4, _dev.ptr(self.tokens), st)
        logits, _ = run_layers(self.model, self.tokens, self.positions, self.n_ctx, self.caches,
                               reuse=self._reuse, logits_rows="last", buffers=self.buffers,
                               timer=self.timer,
                               hook=self._step_hook(hook))
        if logits_out is not None:
            logits_out.copy_(logits, non_blocking=True)
        return logits

    # CUDA graph: one request (copies, selection, 32 layers, logits) replayed
    # with a single launch instead of ~200 host launches ------------------------
    def capture(self, suffix=None, logits_out: torch.Tensor | None = None) -> None:
        """Capture step(suffix, logits_out) into a CUDA graph.  replay() re-runs
        it reading the CURRENT contents of the same suffix/logits buffers."""
        timing, self.timer.enabled = self.timer.enabled, False
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            self.step(suffix, logits_out)          # warm-up: allocations, tables
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        n0 = _lib.LAUNCH_COUNT["n"]
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self._graph_logits = self.step(suffix, logits_out)
        self.launches_per_step = _lib.LAUNCH_COUNT["n"] - n0
        self.timer.enabled = timing

    def replay(self) -> torch.Tensor:
        self.graph.replay()
        _lib.LAUNCH_COUNT["n"] += self.launches_per_step or 0
        return self._graph_logits


class FullPrefillEngine:
    """Full-recompute baseline (ct/toymodel.py:196-205) with the same kernels."""

    def __init__(self, model: GpuModel, n_ctx: int, timer: KernelTimer | None = None):
        cfg = model.config
        dev = model.device
        self.model, self.n_ctx = model, n_ctx
        self.timer = timer or KernelTimer()
        self.cache = torch.empty((cfg.n_layers, 2, n_ctx, cfg.kv_heads, cfg.head_dim),
                                 dtype=model.dtype, device=dev)
        self.caches = [(self.cache[l, 0], self.cache[l, 1]) for l in range(cfg.n_layers)]
        self.buffers = LayerBuffers(model, n_ctx, dev)
        self.positions = torch.arange(n_ctx, dtype=torch.int32, device=dev)

    def attention_flops_per_layer(self) -> float:
        cfg = self.model.config
        n = self.n_ctx
        return 4.0 * cfg.n_heads * cfg.head_dim * n * (n + 1) / 2.0

    def step(self, tokens: torch.Tensor) -> torch.Tensor:
        logits, _ = run_layers(self.model, tokens, self.positions, self.n_ctx, self.caches,
                               logits_rows="last", buffers=self.buffers, timer=self.timer)
        return logits
