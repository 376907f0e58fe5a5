"""(4) Selective-recompute prefill engine (drop-in for ct/toymodel.py:135-311).

`selective_prefill` keeps the reference's signature, validation and result
fields; `full_prefill` is the baseline and r=1 oracle; `encode_chunk_isolated`
produces the pre-RoPE chunk KV (the offline producer).  Per layer the engine
runs (all on the current CUDA stream, every op a libcachetune_b200 kernel;
in the bf16 step the dense projections run on the library's CTA-pair tcgen05
GEMM (ct_gemm_swiglu for gate/up + SwiGLU, ct_gemm_bf16 for QKV / O / down)
where it measured faster, else on cuBLAS via torch.mm):

  K4  ct_qkv_rope_scatter   q,k RoPE at active positions; k,v -> cache rows
  K3  ct_gather_rope_blend  reused rows -> cache rows, K rotated at global pos
  K5  ct_selective_attention  queries = active rows, keys = blended cache
      ct_residual_rmsnorm / ct_mlp_act around the projections.
"""

from __future__ import annotations

import math
import threading
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np
import torch

from . import _dev, _lib
from .errors import InvalidPlan, ShapeError
from .kvcore import DeviceChunk, SeqTensor
from .model import GpuModel
from .rope import rope_table
from .spectral import ImportanceRanking, select_device, selection_count

NORM_EPS = 1e-6  # ct/toymodel.py:28

_models: dict = {}
_models_lock = threading.Lock()


def as_gpu_model(model, dtype=None) -> GpuModel:
    """GpuModel as-is, or a (cached) upload of a reference ToyModel."""
    if isinstance(model, GpuModel):
        return model
    dtype = dtype or torch.float32
    key = (id(model), dtype)
    with _models_lock:
        hit = _models.get(key)
        if hit is not None and hit[0] is model:
            return hit[1]
        dev = _dev.require_cuda()
        g = GpuModel.from_reference(model, dtype=dtype, device=dev)
        _models[key] = (model, g)
        return g


@dataclass(frozen=True)
class AttentionRecord:
    """Per-layer [n_heads, n_queries, n_context] attention (ct/toymodel.py:92-110)."""
    matrices: tuple
    query_positions: np.ndarray
    n_context: int

    def suffix_view(self, suffix_start: int) -> "AttentionRecord":
        rows = np.flatnonzero(self.query_positions >= suffix_start)
        mats = []
        for m in self.matrices:
            if isinstance(m, torch.Tensor):  # device record (record_attention=<position>)
                idx = torch.as_tensor(rows, device=m.device)
                mats.append(m.index_select(1, idx)[:, :, :suffix_start].contiguous())
            else:
                mats.append(np.asarray(m)[:, rows, :suffix_start].copy())
        return AttentionRecord(tuple(mats), self.query_positions[rows].copy(), suffix_start)


def attention_deviation(a: AttentionRecord, b: AttentionRecord) -> float:
    """Mean Frobenius distance of two records (ct/toymodel.py:113-124); device
    records are reduced on the device (f64 accumulation)."""
    if len(a.matrices) != len(b.matrices):
        raise ShapeError("records have different layer counts")
    total, count = 0.0, 0
    for ma, mb in zip(a.matrices, b.matrices):
        if ma.shape != mb.shape:
            raise ShapeError(f"attention shape mismatch {tuple(ma.shape)} vs {tuple(mb.shape)}")
        if isinstance(ma, torch.Tensor) or isinstance(mb, torch.Tensor):
            ta = torch.as_tensor(ma).double()
            tb = torch.as_tensor(mb).to(ta.device).double()
            total += float(torch.linalg.vector_norm(ta - tb, dim=(1, 2)).sum())
            count += ma.shape[0]
            continue
        ma, mb = np.asarray(ma), np.asarray(mb)
        for h in range(ma.shape[0]):
            total += np.linalg.norm(ma[h] - mb[h])
            count += 1
    return float(total / count)


@dataclass
class PrefillResult:
    """ct/toymodel.py:127-132; tensors stay on the device (see to_host)."""
    kv: tuple                  # per layer (K post-RoPE, V), [n_ctx, H_kv, D] tensors
    attention: AttentionRecord | None
    logits: torch.Tensor       # [rows, vocab] f32
    query_positions: np.ndarray

    def to_host(self) -> "PrefillResult":
        kv = tuple((SeqTensor(k.float().cpu().numpy()), SeqTensor(v.float().cpu().numpy()))
                   for k, v in self.kv)
        return PrefillResult(kv, self.attention, self.logits.double().cpu().numpy(),
                             self.query_positions)


def _auto_record(model: GpuModel, a: int, n_ctx: int, record) -> bool:
    if record is not None:
        return bool(record)
    return model.config.n_heads * a * n_ctx <= (1 << 26)


def _record_mode(record):
    """record_attention: None (auto) / bool (every query row, host record) / an
    int position p (device record of the query rows at positions >= p only --
    the suffix rows the quality check reads, ct/toymodel.py:104-110; the main
    attention stays on the tensor-core kernel and the recorded rows are
    recomputed with probabilities by the SIMT kernel)."""
    if isinstance(record, (bool, type(None))):
        return record, None
    return False, int(record)


# CT_MLP_FUSED=0 (read once) keeps the bf16 SwiGLU MLP on cuBLAS + ct_mlp_act
# (the A/B baseline of the fused tcgen05 gate/up kernel)
_MLP_FUSED_ENV = __import__("os").environ.get("CT_MLP_FUSED", "1") != "0"
# row range of the fused kernel (CTA-pair tcgen05 GEMM), from end-to-end A/B
# (tools/mlp_fused_ab.sh, CT_MLP_FUSED=0/1): below 128 rows a tile is mostly
# padding; config 2's 4,992 active rows 95.0 -> 93.1 ms per request, config
# 3's 9,920 rows 256.1 -> 252.6 ms; the 32K / 64K-row full prefill is neutral
# to 0.5 % slower fused (sustained power-capped clocks), so the baseline keeps
# cuBLAS + the activation kernel there and each path runs its faster form
FUSED_MIN_ROWS, FUSED_MAX_ROWS = 128, 16384


def _fused_mlp(model: GpuModel) -> bool:
    """bf16 SwiGLU with tile-friendly widths: gate/up + activation in one
    tcgen05 kernel (ct_gemm_swiglu)."""
    cfg = model.config
    return (_MLP_FUSED_ENV and model.dtype == torch.bfloat16 and cfg.mlp_kind == "swiglu"
            and cfg.hidden_dim % 64 == 0 and cfg.inter % 128 == 0)


class LayerBuffers:
    """Per-run activations (reused across layers)."""

    def __init__(self, model: GpuModel, a: int, dev):
        cfg = model.config
        dt = model.dtype
        hid, d = cfg.hidden_dim, cfg.head_dim
        qkv = (cfg.n_heads + 2 * cfg.kv_heads) * d
        self.h = torch.empty((a, hid), dtype=torch.float32, device=dev)
        self.x = torch.empty((a, hid), dtype=dt, device=dev)
        self.qkv = torch.empty((a, qkv), dtype=dt, device=dev)
        self.q = torch.empty((a, cfg.n_heads, d), dtype=dt, device=dev)
        self.ctx = torch.empty((a, cfg.n_heads * d), dtype=dt, device=dev)
        width = {"relu": 4 * hid, "swiglu": 2 * cfg.inter}.get(cfg.mlp_kind, 0)
        # the bf16 SwiGLU MLP runs fused (ct_gemm_swiglu) for >= FUSED_MIN_ROWS
        # rows, so its [rows, 2I] gate/up buffer only serves smaller calls
        gu_rows = (min(a, FUSED_MIN_ROWS) if cfg.mlp_kind == "swiglu" and _fused_mlp(model)
                   and a <= FUSED_MAX_ROWS else a)
        self.gu = torch.empty((gu_rows, width), dtype=dt, device=dev) if width else None
        self.act = torch.empty((a, width // 2 if cfg.mlp_kind == "swiglu" else width),
                               dtype=dt, device=dev) if width else None


def _mm_f32(a: torch.Tensor, w: torch.Tensor) -> torch.Tensor:
    if a.dtype == torch.float32:
        return torch.mm(a, w)
    return torch.mm(a, w, out_dtype=torch.float32)


# CT_GEMM_OWN=1 (read once) runs the bf16 QKV / O / down projections on
# ct_gemm_bf16 where `_own_gemm` picks it.  Off by default: standalone it is
# up to 19 % faster than cuBLAS, but inside the power-capped step it lowered
# the SM clock (1,470 vs 1,505 MHz) and measured neutral at config 2 (94.9 vs
# 94.9 ms) and 1 % slower at config 3 (261.5 vs 258.8 ms)
_GEMM_OWN_ENV = __import__("os").environ.get("CT_GEMM_OWN", "0") == "1"
# CT_QKV_FUSED=0 (read once): QKV on cuBLAS + the separate ct_qkv_rope_scatter
# epilogue kernel instead of ct_gemm_qkv_rope (A/B switch)
_QKV_FUSED_ENV = __import__("os").environ.get("CT_QKV_FUSED", "1") != "0"
_PAIRS = []


def _own_gemm(a: torch.Tensor, w: torch.Tensor) -> bool:
    """Run a bf16 projection on ct_gemm_bf16 (CTA-pair tcgen05, 256 x 256
    tiles) when its tiles fill >= 90 % of the last wave of the 74 SM pairs,
    else cuBLAS.  tools/gemm_proj_bench.py, ours vs cuBLAS: 9,920 rows (config
    3) QKV / O / down +5 / +11 / +19 % (94-97 % filled); 4,992 rows (config 2)
    QKV +3 % (93 %), O / down -4 / -12 % (320 tiles = 86 % filled, cuBLAS
    kept).  Same row range as the fused MLP."""
    rows, k = a.shape
    n = w.shape[1]
    if not (_GEMM_OWN_ENV and a.dtype == torch.bfloat16 and w.dtype == torch.bfloat16
            and FUSED_MIN_ROWS <= rows <= FUSED_MAX_ROWS and n % 256 == 0 and k % 64 == 0
            and a.stride(1) == 1 and w.stride(1) == 1):
        return False
    if not _PAIRS:
        _PAIRS.append(torch.cuda.get_device_properties(a.device).multi_processor_count // 2)
    tiles = -(-rows // 256) * (n // 256)
    return tiles / (-(-tiles // _PAIRS[0]) * _PAIRS[0]) >= 0.9


def _proj_mm(out: torch.Tensor, a: torch.Tensor, w: torch.Tensor, st) -> None:
    """out = a @ w (the q / k / v projections, ct/toymodel.py:157-159)."""
    if _own_gemm(a, w):
        _lib.call("ct_gemm_bf16", _dev.ptr(a), a.shape[0], a.shape[1], a.stride(0), _dev.ptr(w),
                  w.shape[1], w.stride(0), _dev.ptr(out), out.stride(0), _lib.CT_BF16, 0, st)
    else:
        torch.mm(a, w, out=out)


def _residual_mm(h: torch.Tensor, a: torch.Tensor, w: torch.Tensor, st=None) -> None:
    """h += a @ w in the GEMM epilogue (f32 C/D, bf16 or f32 A/B): the
    residual add of ct/toymodel.py:184,186 without a separate f32 delta round
    trip through HBM.  ct_gemm_bf16 (accumulate) where `_own_gemm` picks it,
    else cuBLAS beta = 1."""
    if a.dtype == torch.float32:
        h.addmm_(a, w)
    elif st is not None and _own_gemm(a, w):
        _lib.call("ct_gemm_bf16", _dev.ptr(a), a.shape[0], a.shape[1], a.stride(0), _dev.ptr(w),
                  w.shape[1], w.stride(0), _dev.ptr(h), h.stride(0), _lib.CT_F32, 1, st)
    else:
        torch.ops.aten.addmm.dtype_out(h, a, w, torch.float32, beta=1, alpha=1, out=h)


def run_layers(model: GpuModel, *args, **kwargs):
    """The fp32 mode promises the 1e-5 tolerance: its cuBLAS GEMMs must not
    silently run as TF32 when a caller enabled that globally, so the flag is
    cleared for the duration of an fp32 run and restored afterwards."""
    flags = torch.backends.cuda.matmul
    if model.dtype != torch.float32 or not flags.allow_tf32:
        return _run_layers(model, *args, **kwargs)
    flags.allow_tf32 = False
    try:
        return _run_layers(model, *args, **kwargs)
    finally:
        flags.allow_tf32 = True


def _run_layers(model: GpuModel, tokens: torch.Tensor, positions: torch.Tensor, n_ctx: int,
                caches: Sequence, reuse: Callable[[int], None] | None = None,
                record_attention: bool = False, logits_rows: str | None = "all",
                k_raw_out: Sequence | None = None, buffers: LayerBuffers | None = None,
                timer=None, hook: Callable[[int, str], None] | None = None,
                record_rows_from: int | None = None, prune_last: bool = True):
    """Shared forward engine (ct/toymodel.py:135-193) over device inputs.

    tokens/positions: int32 [A] device.  caches[l] = (K, V) [n_ctx, Hkv, D]
    (model dtype).  reuse(l) fills the reused rows of layer l before its
    attention.  record_rows_from=i records probabilities of query rows [i, A)
    only.  prune_last: with logits_rows "last" / None the last layer's
    attention and MLP run on the last row only / are skipped (the caches are
    complete either way).  Returns (logits f32 [rows, V] or None, probs list)."""
    cfg = model.config
    dev = model.device
    a = tokens.numel()
    hid, hq, hkv, d = cfg.hidden_dim, cfg.n_heads, cfg.kv_heads, cfg.head_dim
    dt = model.dtype
    dtc = _dev.ct_dtype(dt)
    st = _dev.stream_handle()
    lib = _lib.load()
    buf = buffers or LayerBuffers(model, a, dev)
    n_layers = len(model.layers)
    params = cfg.rope_params
    table = rope_table(params, n_ctx, "f64" if dt == torch.float32 else "f32", dev)
    wsb = lib.ct_attention_workspace_bytes(a, hq, n_ctx, hkv, d, dtc)
    ws = _dev.workspace(wsb, "attention")
    scale = 1.0 / math.sqrt(d)
    # bf16 / head_dim 128 / adjacent pairs: q|k|v GEMM with RoPE + cache
    # scatter in its epilogue (ct_gemm_qkv_rope) over the fused-MLP row range.
    # Standalone it is 1.09-1.48x over cuBLAS + ct_qkv_rope_scatter from 2,048
    # to 65,600 rows (profiles/round2_qkv_rows.txt), but inside the
    # power-capped 32K-row full prefill it measured 0.8 % slower
    # (profiles/round2_qkv_full_ab.txt), so, like the MLP, each path runs its
    # faster form
    qkv_fused = (_QKV_FUSED_ENV and dt == torch.bfloat16 and d == 128 and not k_raw_out
                 and params.pairing_code == _lib.CT_ROPE_ADJACENT
                 and FUSED_MIN_ROWS <= a <= FUSED_MAX_ROWS and (hq + 2 * hkv) % 2 == 0
                 and hid % 64 == 0 and buf.x.stride(1) == 1
                 and all(lw["wqkv"].stride(1) == 1 for lw in model.layers))
    _lib.call("ct_embedding_gather", _dev.ptr(model.embedding), _dev.ptr(tokens), a, hid,
              _dev.ptr(buf.h), st)
    _lib.call("ct_residual_rmsnorm", _dev.ptr(buf.h), None, _lib.CT_F32, a, hid, NORM_EPS,
              _dev.ptr(buf.x), dtc, st)
    probs_all = []
    for l, w in enumerate(model.layers):
        kc, vc = caches[l]
        if hook is not None:
            hook(l, "start")
        if qkv_fused:
            wq = w["wqkv"]
            tq = timer.start("qkv_gemm") if timer is not None else None
            _lib.call("ct_gemm_qkv_rope", _dev.ptr(buf.x), a, hid, buf.x.stride(0), _dev.ptr(wq),
                      wq.stride(0), _dev.ptr(positions), _dev.ptr(table), hq, hkv, d,
                      _dev.ptr(buf.q), _dev.ptr(kc), _dev.ptr(vc), hkv * d, st)
            if timer is not None:
                timer.stop("qkv_gemm", tq)
        else:
            _proj_mm(buf.qkv, buf.x, w["wqkv"], st)
            tq = timer.start("qkv") if timer is not None else None
            _lib.check(lib.ct_qkv_rope_scatter(
                _dev.ptr(buf.qkv), buf.qkv.shape[1], dtc, _dev.ptr(positions), a, hq, hkv, d,
                params.pairing_code, _dev.ptr(table), _dev.ptr(buf.q), dtc, _dev.ptr(kc),
                _dev.ptr(vc), dtc, hkv * d, _dev.ptr(k_raw_out[l]) if k_raw_out else None, st),
                "ct_qkv_rope_scatter")
            if timer is not None:
                timer.stop("qkv", tq)
        if hook is not None:
            hook(l, "recomputed")
        if reuse is not None:
            reuse(l)
        # Last layer: once its K/V rows are in the cache nothing downstream
        # reads the other rows' outputs, so when only the first-token logits
        # (or nothing) are wanted, attention / O-projection / MLP run on the
        # last row alone (or are skipped).  Recording keeps every row.
        r0 = 0
        if l == n_layers - 1 and prune_last and not record_attention and record_rows_from is None:
            if logits_rows is None:
                if hook is not None:
                    hook(l, "end")
                break
            if logits_rows != "all":
                r0 = a - 1
        av = a - r0
        hv, xv, qv, ctxv, posv = buf.h[r0:], buf.x[r0:], buf.q[r0:], buf.ctx[r0:], positions[r0:]
        if r0:  # few-row (split-key) attention: its own workspace
            wsb = lib.ct_attention_workspace_bytes(av, hq, n_ctx, hkv, d, dtc)
            ws = _dev.workspace(wsb, "attention_rows")
        probs = (torch.empty((hq, a, n_ctx), dtype=torch.float32, device=dev)
                 if record_attention else None)
        tname = "attention" if r0 == 0 else "attention_last_row"
        t0 = timer.start(tname) if timer is not None else None
        _lib.check(lib.ct_selective_attention(
            _dev.ptr(qv), _dev.ptr(posv), av, hq, _dev.ptr(kc), _dev.ptr(vc), n_ctx, hkv,
            d, kc.stride(0), scale, dtc, _dev.ptr(ctxv), dtc, _dev.ptr(probs), _dev.ptr(ws),
            wsb, st), "ct_selective_attention")
        if timer is not None:
            timer.stop(tname, t0)
        if record_attention:
            probs_all.append(probs)
        elif record_rows_from is not None and record_rows_from < a:
            nr = a - record_rows_from
            part = torch.empty((hq, nr, n_ctx), dtype=torch.float32, device=dev)
            scratch = torch.empty((nr, hq * d), dtype=dt, device=dev)
            wsr = lib.ct_attention_workspace_bytes(nr, hq, n_ctx, hkv, d, dtc)
            _lib.check(lib.ct_selective_attention(
                _dev.ptr(buf.q[record_rows_from:]), _dev.ptr(positions[record_rows_from:]), nr,
                hq, _dev.ptr(kc), _dev.ptr(vc), n_ctx, hkv, d, kc.stride(0), scale, dtc,
                _dev.ptr(scratch), dtc, _dev.ptr(part), _dev.ptr(_dev.workspace(wsr, "record")),
                wsr, st), "ct_selective_attention")
            probs_all.append(part)
        _residual_mm(hv, ctxv, w["wo"], st)
        _lib.call("ct_residual_rmsnorm", _dev.ptr(hv), None, _lib.CT_F32, av, hid,
                  NORM_EPS, _dev.ptr(xv), dtc, st)
        kind = cfg.mlp_kind
        if kind:
            up = w["w1"] if kind == "relu" else w["wgu"]
            down = w["w2"] if kind == "relu" else w["wd"]
            actv = buf.act[r0:]
            inter = buf.act.shape[1]
            if (kind == "swiglu" and FUSED_MIN_ROWS <= av <= FUSED_MAX_ROWS
                    and _fused_mlp(model)):
                tg = timer.start("mlp_gemm") if timer is not None else None
                _lib.call("ct_gemm_swiglu", _dev.ptr(xv), av, hid, xv.stride(0), _dev.ptr(up),
                          inter, up.stride(0), _dev.ptr(actv), actv.stride(0), st)
                if timer is not None:
                    timer.stop("mlp_gemm", tg)
            else:
                guv = buf.gu[:av]
                torch.mm(xv, up, out=guv)
                _lib.call("ct_mlp_act", _dev.ptr(guv), av, inter, dtc,
                          1 if kind == "relu" else 0, _dev.ptr(actv), dtc, st)
            _residual_mm(hv, actv, down, st)
            _lib.call("ct_residual_rmsnorm", _dev.ptr(hv), None, _lib.CT_F32, av,
                      hid, NORM_EPS, _dev.ptr(xv), dtc, st)
        if hook is not None:
            hook(l, "end")
    logits = None
    if logits_rows is not None and a:
        hrows = buf.h if logits_rows == "all" else buf.h[-1:]
        logits = _mm_f32(hrows.to(model.w_out.dtype), model.w_out)
    return logits, probs_all


def _check_tokens(model: GpuModel, toks: np.ndarray) -> None:
    """ct/toymodel.py:81-85."""
    if toks.ndim != 1 or toks.size < 1:
        raise ShapeError("token ids must be a non-empty 1-d array")
    if toks.min() < 0 or toks.max() >= model.config.vocab_size:
        raise ShapeError("token id out of vocabulary")


def _new_caches(model: GpuModel, n_ctx: int, dev):
    cfg = model.config
    return [(torch.empty((n_ctx, cfg.kv_heads, cfg.head_dim), dtype=model.dtype, device=dev),
             torch.empty((n_ctx, cfg.kv_heads, cfg.head_dim), dtype=model.dtype, device=dev))
            for _ in range(cfg.n_layers)]


def full_prefill(model, tokens: Sequence[int], *, record_attention=None,
                 logits_rows: str = "all", dtype=None) -> PrefillResult:
    """Standard causal forward over the whole prompt (ct/toymodel.py:196-205)."""
    g = as_gpu_model(model, dtype)
    toks = np.asarray(tokens, dtype=np.int64)
    _check_tokens(g, toks)
    dev = g.device
    n = toks.size
    tok_d = torch.as_tensor(toks.astype(np.int32), device=dev)
    pos_d = torch.arange(n, dtype=torch.int32, device=dev)
    caches = _new_caches(g, n, dev)
    rec, rows_from = _record_mode(record_attention)
    if rows_from is not None:
        rows_from = min(max(rows_from, 0), n)
        logits, probs = run_layers(g, tok_d, pos_d, n, caches, logits_rows=logits_rows,
                                   record_rows_from=rows_from)
        att = AttentionRecord(tuple(probs), np.arange(rows_from, n), n)
        return PrefillResult(tuple(caches), att, logits, np.arange(n))
    rec = _auto_record(g, n, n, rec)
    logits, probs = run_layers(g, tok_d, pos_d, n, caches, record_attention=rec,
                               logits_rows=logits_rows)
    att = (AttentionRecord(tuple(p.cpu().numpy() for p in probs), np.arange(n), n)
           if rec else None)
    return PrefillResult(tuple(caches), att, logits, np.arange(n))


def encode_chunk_isolated(model, tokens: Sequence[int], chunk_id: str = "chunk", *,
                          dtype=None, out=None) -> DeviceChunk:
    """Forward the chunk alone at local positions; keep pre-RoPE K (ct/toymodel.py:208-220).

    out=(keys, values): contiguous [L, N, Hkv, D] device tensors of the model
    dtype the layers write into (e.g. one chunk's slice of the offline stage's
    [C, L, N, Hkv, D] scorer batch), instead of fresh allocations."""
    g = as_gpu_model(model, dtype)
    toks = np.asarray(tokens, dtype=np.int64)
    _check_tokens(g, toks)
    cfg = g.config
    dev = g.device
    n = toks.size
    shape = (cfg.n_layers, n, cfg.kv_heads, cfg.head_dim)
    if out is None:
        keys = torch.empty(shape, dtype=g.dtype, device=dev)
        vals = torch.empty(shape, dtype=g.dtype, device=dev)
    else:
        keys, vals = out
        for t in (keys, vals):
            if tuple(t.shape) != shape or t.dtype != g.dtype or not t.is_contiguous() \
                    or t.device != torch.device(dev):
                raise ShapeError(f"out tensors must be contiguous {shape} {g.dtype} on {dev}")
    krot = torch.empty(shape[1:], dtype=g.dtype, device=dev)
    caches = [(krot, vals[l]) for l in range(cfg.n_layers)]
    tok_d = torch.as_tensor(toks.astype(np.int32), device=dev)
    pos_d = torch.arange(n, dtype=torch.int32, device=dev)
    run_layers(g, tok_d, pos_d, n, caches, logits_rows=None,
               k_raw_out=[keys[l] for l in range(cfg.n_layers)])
    return DeviceChunk(chunk_id, keys, vals, tok_d, toks)


def _validate(cfg, chunks, rankings):
    """ct/toymodel.py:234-244."""
    if len(chunks) == 0 or len(chunks) != len(rankings):
        raise InvalidPlan("need one ranking per chunk")
    for chunk, ranking in zip(chunks, rankings):
        if ranking.n_tokens != chunk.token_count:
            raise InvalidPlan("ranking/chunk token counts disagree")
        if chunk.n_layers != cfg.n_layers:
            raise InvalidPlan("chunk layer count disagrees with model")
        if (chunk.n_heads, chunk.head_dim) != (cfg.kv_heads, cfg.head_dim):
            raise ShapeError("chunk geometry disagrees with model")
        if chunk.source_tokens is None:
            raise InvalidPlan("chunk lacks source_tokens; cannot recompute")


def selective_prefill(model, chunks: Sequence, rankings: Sequence, suffix_tokens: Sequence[int],
                      r: float, *, record_attention=None, logits_rows: str = "all",
                      dtype=None) -> PrefillResult:
    """Online reuse path (ct/toymodel.py:223-311): recompute the ratio-r
    selection plus the suffix; every other token contributes its reused KV
    through deferred-RoPE scatter fusion.  At r=1 this reproduces full_prefill."""
    g = as_gpu_model(model, dtype)
    cfg = g.config
    _validate(cfg, chunks, rankings)
    # host-side selection (ct/toymodel.py:246-267) so the active token ids are
    # validated before any device work (ct/toymodel.py:303), as the reference
    # does, and the query positions need no device readback later
    sizes = [c.token_count for c in chunks]
    offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    suffix = np.asarray(suffix_tokens, dtype=np.int64)
    ks_host = [selection_count(r, n) for n in sizes]
    rec_host = np.sort(np.concatenate(
        [np.asarray(rk.aggregate_order[:k], np.int64) + off
         for rk, k, off in zip(rankings, ks_host, offsets)] or [np.empty(0, np.int64)]))
    src_host = np.concatenate([np.asarray(c.source_tokens, np.int64) for c in chunks])
    qpos_host = np.concatenate([rec_host, np.arange(offsets[-1], offsets[-1] + suffix.size)])
    if qpos_host.size:
        _check_tokens(g, np.concatenate([src_host[rec_host], suffix]))
    dev = g.device
    dchunks = [c if isinstance(c, DeviceChunk) else DeviceChunk.from_host(c, g.dtype, dev)
               for c in chunks]
    for c in dchunks:
        if c.keys.dtype != g.dtype:
            raise ShapeError(f"chunk dtype {c.keys.dtype} != model dtype {g.dtype}")
    history = int(offsets[-1])
    n_ctx = history + suffix.size
    aggs = [rk.aggregate_device(dev) if isinstance(rk, ImportanceRanking)
            else torch.as_tensor(np.asarray(rk.aggregate_order, np.int32), device=dev)
            for rk in rankings]
    rec, keep, _, ks = select_device(aggs, r, dev)
    n_rec = rec.numel()
    # active tokens = source tokens of the recomputed rows, then the suffix
    src_all = torch.cat([c.tokens if c.tokens is not None else
                         torch.as_tensor(np.asarray(c.source_tokens, np.int32), device=dev)
                         for c in dchunks])
    a = n_rec + suffix.size
    positions = torch.empty(a, dtype=torch.int32, device=dev)
    tokens = torch.empty(a, dtype=torch.int32, device=dev)
    positions[:n_rec] = rec
    if suffix.size:
        positions[n_rec:] = torch.arange(history, n_ctx, dtype=torch.int32, device=dev)
        tokens[n_rec:] = torch.as_tensor(suffix.astype(np.int32), device=dev)
    if n_rec:
        _lib.call("ct_gather_rows", _dev.ptr(src_all), _dev.ptr(rec), n_rec, 4,
                  _dev.ptr(tokens), _dev.stream_handle())
    caches = _new_caches(g, n_ctx, dev)
    hkv, d = cfg.kv_heads, cfg.head_dim
    keep_base = np.concatenate([[0], np.cumsum([n - k for n, k in zip(sizes, ks)])])
    table = rope_table(cfg.rope_params, max(n_ctx, 1), "f64" if g.dtype == torch.float32
                       else "f32", dev)
    esize = torch.empty((), dtype=g.dtype).element_size()

    def reuse(l: int) -> None:
        segs = []
        for j, c in enumerate(dchunks):
            nk = int(keep_base[j + 1] - keep_base[j])
            if nk == 0:
                continue
            # src row = global token - chunk offset: shift the base pointer
            shift = int(offsets[j]) * hkv * d * esize
            segs.append(_lib.Segment(_dev.ptr(c.keys[l]) - shift, _dev.ptr(c.values[l]) - shift,
                                     _dev.ptr(keep) + int(keep_base[j]) * 4, nk, 0, 1))
        kc, vc = caches[l]
        for s0 in range(0, len(segs), _lib.CT_MAX_SEGMENTS):
            part = segs[s0:s0 + _lib.CT_MAX_SEGMENTS]
            arr = (_lib.Segment * len(part))(*part)
            _lib.call("ct_gather_rope_blend", arr, len(part), hkv * d, hkv, d,
                      _dev.ct_dtype(g.dtype), cfg.rope_params.pairing_code, _dev.ptr(table),
                      _dev.ptr(kc), _dev.ptr(vc), hkv * d, _dev.stream_handle())

    if a == 0:
        for l in range(cfg.n_layers):
            reuse(l)
        att = AttentionRecord(tuple(np.zeros((cfg.n_heads, 0, n_ctx)) for _ in range(cfg.n_layers)),
                              np.empty(0, np.int64), n_ctx)
        return PrefillResult(tuple(caches), att,
                             torch.zeros((0, cfg.vocab_size), dtype=torch.float32, device=dev),
                             np.empty(0, np.int64))
    rec_attn, rec_pos = _record_mode(record_attention)
    if rec_pos is not None:
        rows_from = int(np.searchsorted(qpos_host, rec_pos, side="left"))
        logits, probs = run_layers(g, tokens, positions, n_ctx, caches, reuse=reuse,
                                   logits_rows=logits_rows, record_rows_from=rows_from)
        att = AttentionRecord(tuple(probs), qpos_host[rows_from:].copy(), n_ctx)
        return PrefillResult(tuple(caches), att, logits, qpos_host)
    rec_attn = _auto_record(g, a, n_ctx, rec_attn)
    logits, probs = run_layers(g, tokens, positions, n_ctx, caches, reuse=reuse,
                               record_attention=rec_attn, logits_rows=logits_rows)
    att = (AttentionRecord(tuple(p.cpu().numpy() for p in probs), qpos_host, n_ctx)
           if rec_attn else None)
    return PrefillResult(tuple(caches), att, logits, qpos_host)
