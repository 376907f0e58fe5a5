"""(1) Frequency-domain critical-token scorer and ratio selection.

Drop-in for ct/spectral.py: same names, argument order, defaults and errors.
The arithmetic runs in libcachetune_b200.so (ct_score_chunks /
ct_desc_order / ct_selection_plan); host code only validates arguments and
moves results.  `precision="f64"` (default) scores with a float64 FFT like the
reference's pocketfft so per-layer and aggregate orders are bit-exact;
"f32" is the fast mode.
"""

from __future__ import annotations

import ctypes

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _dev, _lib
from .errors import InvalidParam, ShapeError
from .kvcore import ComplexSpectrum, DeviceChunk, KvChunk, SeqTensor

DEFAULT_ALPHA = 0.5  # ct/spectral.py:24


def cutoff_index(alpha: float, n_freqs: int) -> int:
    """c = floor(alpha * n_freqs) as a float product (ct/spectral.py:57-58)."""
    return int(math.floor(alpha * n_freqs))


def _check_alpha(alpha: float) -> None:
    if not 0.0 <= alpha <= 1.0:
        raise InvalidParam(f"alpha must be in [0, 1], got {alpha}")


def selection_count(r: float, n_tokens: int) -> int:
    """ceil(r*N - 1e-9) clamped to [0, N] (ct/spectral.py:162-172)."""
    if not 0.0 <= r <= 1.0:
        raise InvalidParam(f"ratio must be in [0, 1], got {r}")
    k = math.ceil(r * n_tokens - 1e-9)
    return min(max(k, 0), n_tokens)


@dataclass(frozen=True)
class ImportanceRanking:
    """Descending token permutations (ct/spectral.py:104-146).

    Host arrays as in the reference; `device_aggregate` (optional) keeps the
    aggregate order resident in HBM as int32 for the online path."""

    per_layer_scores: np.ndarray
    per_layer_order: np.ndarray
    aggregate_order: np.ndarray
    alpha: float
    n_tokens: int
    device_aggregate: object = None

    def __post_init__(self):
        scores = np.asarray(self.per_layer_scores, dtype=np.float64)
        orders = np.asarray(self.per_layer_order, dtype=np.int64)
        agg = np.asarray(self.aggregate_order, dtype=np.int64)
        if scores.ndim != 2 or scores.shape != orders.shape:
            raise ShapeError("per-layer scores/orders must be [L, N] and congruent")
        n = self.n_tokens
        if scores.shape[1] != n or agg.shape != (n,):
            raise ShapeError("ranking arrays disagree with n_tokens")
        want = np.arange(n)
        if not np.array_equal(np.sort(agg), want):
            raise InvalidParam("aggregate_order is not a permutation of [0, N)")
        for row in orders:
            if not np.array_equal(np.sort(row), want):
                raise InvalidParam("per-layer order is not a permutation of [0, N)")
        if not np.all(np.isfinite(scores)) or (scores.size and scores.min() < 0):
            raise InvalidParam("scores must be finite and >= 0")
        for name, arr in (("per_layer_scores", scores), ("per_layer_order", orders),
                          ("aggregate_order", agg)):
            arr = np.ascontiguousarray(arr)
            arr.flags.writeable = False
            object.__setattr__(self, name, arr)

    @property
    def n_layers(self) -> int:
        return self.per_layer_scores.shape[0]

    def aggregate_device(self, device) -> torch.Tensor:
        d = self.device_aggregate
        if d is not None and d.device == torch.device(device):
            return d
        return torch.as_tensor(self.aggregate_order.astype(np.int32), device=device)


def _as_device_kv(keys, values):
    """Accept SeqTensor-likes, numpy [N,H,D] or torch tensors [L?,N,H,D]."""
    dev = _dev.require_cuda()

    def conv(x):
        if isinstance(x, torch.Tensor):
            return x.to(dev)
        data = x.data if hasattr(x, "data") and not isinstance(x, np.ndarray) else x
        arr = np.ascontiguousarray(np.asarray(data, dtype=np.float32))
        if not arr.flags.writeable:  # SeqTensor data is frozen; torch wants writable
            arr = arr.copy()
        return torch.from_numpy(arr).to(dev)
    k, v = conv(keys), conv(values)
    if k.dim() == 3:
        k, v = k.unsqueeze(0), v.unsqueeze(0)
    return k, v


def score_device(keys: torch.Tensor, values: torch.Tensor, alpha: float = DEFAULT_ALPHA,
                 precision: str = "f64", want_layer_order: bool = True, band: str = "low",
                 out: dict | None = None):
    """Score C chunks on the device (band "low", or "high" = ct/spectral.py:47-54).

    keys/values: [C, L, N, H, D] (or [L, N, H, D]) f32/bf16 CUDA tensors.
    Returns dict of device tensors: layer_scores [C,L,N] f64, agg [C,N] f64,
    layer_order [C,L,N] int32 (optional), agg_order [C,N] int32.  `out`: the
    same dict of caller-allocated contiguous tensors to write into (e.g. one
    chunk's slices of a batch result)."""
    _check_alpha(alpha)
    if band not in ("low", "high"):
        raise InvalidParam(f"band must be 'low' or 'high', got {band!r}")
    if keys.shape != values.shape:
        raise ShapeError(f"keys {tuple(keys.shape)} vs values {tuple(values.shape)}")
    if keys.dim() == 4:
        keys, values = keys.unsqueeze(0), values.unsqueeze(0)
    if keys.dim() != 5:
        raise ShapeError("expected [C, L, N, H, D]")
    keys, values = keys.contiguous(), values.contiguous()
    C, L, N, H, D = keys.shape
    lanes = H * D
    dev = keys.device
    cutoff = cutoff_index(alpha, N // 2 + 1)
    prec = _lib.CT_F64 if precision == "f64" else _lib.CT_F32
    shapes = {"layer_scores": ((C, L, N), torch.float64), "agg": ((C, N), torch.float64),
              "agg_order": ((C, N), torch.int32), "layer_order": ((C, L, N), torch.int32)}
    if out is None:
        out = {k: torch.empty(sh, dtype=dt, device=dev) for k, (sh, dt) in shapes.items()}
        if not want_layer_order:
            out["layer_order"] = None
    else:
        for k, (sh, dt) in shapes.items():
            t = out.get(k)
            if t is None and k == "layer_order" and not want_layer_order:
                continue
            if t is None or tuple(t.shape) != sh or t.dtype != dt or not t.is_contiguous() \
                    or t.device != dev:
                raise ShapeError(f"out[{k!r}] must be a contiguous {sh} {dt} tensor on {dev}")
    lib = _lib.load()
    wsb = lib.ct_score_workspace_bytes(C, L, N, lanes, prec)
    ws = _dev.workspace(wsb, "score")
    _lib.check(lib.ct_score_chunks_band(
        _dev.ptr(keys), _dev.ptr(values), _dev.ct_dtype(keys.dtype), C, L, N, lanes,
        lanes, N * lanes, L * N * lanes, cutoff, prec, 1 if band == "high" else 0,
        _dev.ptr(out["layer_scores"]), _dev.ptr(out["agg"]), _dev.ptr(out["layer_order"]),
        _dev.ptr(out["agg_order"]), _dev.ptr(ws), wsb, _dev.stream_handle()),
        "ct_score_chunks_band")
    return out


# Relative error bound of the single-precision aggregate scores of
# ct_score_select_fast (calibrated on model-encoded and Gaussian chunks,
# DESIGN.md "Fast scorer"), and the widest boundary window re-scored on the
# device (wider windows fall back to the exact scorer for that chunk).
FAST_GUARD = 2e-6
FAST_WMAX = 64


def score_select_fast(keys: torch.Tensor, values: torch.Tensor, k: int,
                      alpha: float = DEFAULT_ALPHA, guard: float = FAST_GUARD,
                      band: str = "low", want_layer_scores: bool = False):
    """Scores + an aggregate order whose first k entries are exactly the
    float64 top-k set (ct/spectral.py:149-178), from single-precision FFTs
    (ct_score_select_fast).  keys/values [C, L, 2048, H, D] (or [L, ...]) on
    the device; H*D a multiple of 128.  Chunks whose boundary window is wider
    than FAST_WMAX are re-scored with the exact float64 scorer (their whole
    order is then exact).  Returns device tensors agg [C,N] f64, agg_order
    [C,N] int32, wcount [C] int32 (0 = certified by the guard, w = w tokens
    re-scored, -1 = exact fallback) and layer_scores [C,L,N] (or None)."""
    _check_alpha(alpha)
    if band not in ("low", "high"):
        raise InvalidParam(f"band must be 'low' or 'high', got {band!r}")
    if keys.shape != values.shape:
        raise ShapeError(f"keys {tuple(keys.shape)} vs values {tuple(values.shape)}")
    if keys.dim() == 4:
        keys, values = keys.unsqueeze(0), values.unsqueeze(0)
    if keys.dim() != 5:
        raise ShapeError("expected [C, L, N, H, D]")
    keys, values = keys.contiguous(), values.contiguous()
    C, L, N, H, D = keys.shape
    if not 0 <= k <= N:
        raise InvalidParam(f"k must be in [0, {N}], got {k}")
    lanes = H * D
    dev = keys.device
    cutoff = cutoff_index(alpha, N // 2 + 1)
    lib = _lib.load()
    wsb = lib.ct_score_fast_workspace_bytes(C, L, N, lanes)
    if wsb == 0:
        raise _lib.Unsupported(f"fast scorer needs N = 2048 and H*D % 128 == 0 (N={N})")
    out = {
        "agg": torch.empty((C, N), dtype=torch.float64, device=dev),
        "agg_order": torch.empty((C, N), dtype=torch.int32, device=dev),
        "wcount": torch.empty(C, dtype=torch.int32, device=dev),
        "layer_scores": (torch.empty((C, L, N), dtype=torch.float64, device=dev)
                         if want_layer_scores else None),
    }
    ws = _dev.workspace(wsb, "score_fast")
    _lib.check(lib.ct_score_select_fast(
        _dev.ptr(keys), _dev.ptr(values), _dev.ct_dtype(keys.dtype), C, L, N, lanes, lanes,
        N * lanes, L * N * lanes, cutoff, 1 if band == "high" else 0, k, guard,
        _dev.ptr(out["layer_scores"]), _dev.ptr(out["agg"]), _dev.ptr(out["agg_order"]),
        _dev.ptr(out["wcount"]), _dev.ptr(ws), wsb, _dev.stream_handle()),
        "ct_score_select_fast")
    wide = torch.nonzero(out["wcount"] > FAST_WMAX).flatten().tolist()
    if wide:  # pathological windows (ties, near-constant chunks): exact scorer
        sel = torch.as_tensor(wide, device=dev)
        ex = score_device(keys.index_select(0, sel), values.index_select(0, sel), alpha, "f64",
                          want_layer_order=False, band=band)
        out["agg"][sel] = ex["agg"]
        out["agg_order"][sel] = ex["agg_order"]
        if out["layer_scores"] is not None:
            out["layer_scores"][sel] = ex["layer_scores"]
        out["wcount"][sel] = -1
    return out


def low_freq_scores(keys, values, alpha: float = DEFAULT_ALPHA,
                    precision: str = "f64") -> np.ndarray:
    """Per-token importance (ct/spectral.py:82-90): 0.5|K~_i| + 0.5|V~_i|."""
    _check_alpha(alpha)
    ks = getattr(keys, "shape", None)
    vs = getattr(values, "shape", None)
    if tuple(ks) != tuple(vs):
        raise ShapeError(f"keys {ks} vs values {vs}")
    k, v = _as_device_kv(keys, values)
    out = score_device(k, v, alpha, precision, want_layer_order=False)
    return out["layer_scores"][0, 0].cpu().numpy()


def high_freq_scores(keys, values, alpha: float = DEFAULT_ALPHA,
                     precision: str = "f64") -> np.ndarray:
    """Mirror of low_freq_scores on the complementary high band (ct/spectral.py:93-96)."""
    _check_alpha(alpha)
    ks = getattr(keys, "shape", None)
    vs = getattr(values, "shape", None)
    if tuple(ks) != tuple(vs):
        raise ShapeError(f"keys {ks} vs values {vs}")
    k, v = _as_device_kv(keys, values)
    out = score_device(k, v, alpha, precision, want_layer_order=False, band="high")
    return out["layer_scores"][0, 0].cpu().numpy()


def _chunk_tensors(chunk):
    if isinstance(chunk, DeviceChunk):
        return chunk.keys, chunk.values
    dev = _dev.require_cuda()
    k = np.stack([np.asarray(t.data, dtype=np.float32) for t in chunk.keys_raw])
    v = np.stack([np.asarray(t.data, dtype=np.float32) for t in chunk.values])
    return torch.from_numpy(k).to(dev), torch.from_numpy(v).to(dev)


def rank_chunk(chunk, alpha: float = DEFAULT_ALPHA, precision: str = "f64",
               band: str = "low") -> ImportanceRanking:
    """Score every layer and build the importance permutations (ct/spectral.py:149-159;
    band="high" is the highfreq strategy's ranking, ct/toymodel.py:356-363)."""
    _check_alpha(alpha)
    k, v = _chunk_tensors(chunk)
    out = score_device(k, v, alpha, precision, band=band)
    n = k.shape[1]
    return ImportanceRanking(
        per_layer_scores=out["layer_scores"][0].cpu().numpy(),
        per_layer_order=out["layer_order"][0].cpu().numpy().astype(np.int64),
        aggregate_order=out["agg_order"][0].cpu().numpy().astype(np.int64),
        alpha=alpha, n_tokens=n, device_aggregate=out["agg_order"][0])


def rank_chunks(chunks, alpha: float = DEFAULT_ALPHA, precision: str = "f64",
                host: bool = True):
    """Batched rank_chunk over equal-geometry device chunks (one launch set)."""
    keys = torch.stack([c.keys for c in chunks])
    vals = torch.stack([c.values for c in chunks])
    out = score_device(keys, vals, alpha, precision, want_layer_order=host)
    if not host:
        return out
    res = []
    ls, lo, ao = (out["layer_scores"].cpu().numpy(), out["layer_order"].cpu().numpy(),
                  out["agg_order"].cpu().numpy())
    for i in range(len(chunks)):
        res.append(ImportanceRanking(per_layer_scores=ls[i], per_layer_order=lo[i].astype(np.int64),
                                     aggregate_order=ao[i].astype(np.int64), alpha=alpha,
                                     n_tokens=keys.shape[2], device_aggregate=out["agg_order"][i]))
    return res


def select_device(agg_orders: list, ratios, device=None):
    """Device selection plan over chunks laid end to end (ct/spectral.py:175-184,
    ct/toymodel.py:246-260).  agg_orders: list of device int32 [N_j] tensors.
    Returns (rec_global int32 ascending, keep_global int32 ascending,
    keep_src_row int32 importance ranks, ks list)."""
    device = device or agg_orders[0].device
    if np.isscalar(ratios):
        ratios = [ratios] * len(agg_orders)
    sizes = [int(a.numel()) for a in agg_orders]
    ks = [selection_count(r, n) for r, n in zip(ratios, sizes)]
    offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    rec_base = np.concatenate([[0], np.cumsum(ks)]).astype(np.int64)
    keep_base = np.concatenate([[0], np.cumsum([n - k for n, k in zip(sizes, ks)])]).astype(np.int64)
    meta = torch.as_tensor(np.concatenate([offsets, np.asarray(ks, np.int64), rec_base,
                                           keep_base]), device=device)
    nc = len(sizes)
    off_d = meta[: nc + 1]
    ks_d = meta[nc + 1: 2 * nc + 1]
    rb_d = meta[2 * nc + 1: 3 * nc + 2]
    kb_d = meta[3 * nc + 2:]
    aggs = torch.cat([a.to(torch.int32) for a in agg_orders])
    rec = torch.empty(int(rec_base[-1]), dtype=torch.int32, device=device)
    keep = torch.empty(int(keep_base[-1]), dtype=torch.int32, device=device)
    ksrc = torch.empty_like(keep)
    _lib.call("ct_selection_plan", _dev.ptr(aggs), _dev.ptr(off_d), _dev.ptr(ks_d),
              _dev.ptr(rb_d), _dev.ptr(kb_d), nc, max(sizes), _dev.ptr(rec), _dev.ptr(keep),
              _dev.ptr(ksrc), _dev.stream_handle())
    return rec, keep, ksrc, ks


def _select_one(ranking, r: float):
    """ct_select on one ranking: (selected ascending, kept ascending) int32 on
    the device, k computed by the C ABI with the reference's guard."""
    n = int(ranking.n_tokens)
    k = selection_count(r, n)  # validates r (InvalidParam before any work)
    dev = _dev.require_cuda()
    agg = (ranking.aggregate_device(dev) if isinstance(ranking, ImportanceRanking)
           else torch.as_tensor(np.asarray(ranking.aggregate_order, np.int32), device=dev))
    agg = agg.to(torch.int32).contiguous()
    sel = torch.empty(k, dtype=torch.int32, device=dev)
    keep = torch.empty(n - k, dtype=torch.int32, device=dev)
    k_abi = ctypes.c_int64(-1)
    _lib.call("ct_select", _dev.ptr(agg), n, float(r), _dev.ptr(sel), _dev.ptr(keep),
              ctypes.addressof(k_abi), _dev.stream_handle())
    if k_abi.value != k:  # pragma: no cover - the two restatements must agree
        raise RuntimeError(f"ct_select k={k_abi.value}, selection_count={k}")
    return sel, keep


def indices_for_ratio(ranking, r: float) -> np.ndarray:
    """First ceil(r*N) tokens of the aggregate order, ascending (ct/spectral.py:175-178)."""
    sel, _ = _select_one(ranking, r)
    return sel.cpu().numpy().astype(np.int64)


def complement_for_ratio(ranking, r: float) -> np.ndarray:
    """Tokens NOT selected at ratio r, ascending (ct/spectral.py:181-184)."""
    _, keep = _select_one(ranking, r)
    return keep.cpu().numpy().astype(np.int64)


# -- spectrum building blocks (ct/spectral.py:27-66) and selection diagnostics
# (:187-208).  Analysis helpers, NOT the scoring path: low_freq_scores /
# rank_chunk run the fused FFT -> band mask -> inverse FFT -> energy kernel
# and never materialise a spectrum.  The transforms here are cuFFT (torch.fft)
# in float64 on the device, the same role spectrum_report gives them.

def _seq_device(t) -> torch.Tensor:
    if isinstance(t, torch.Tensor):
        return t.to(torch.float64)
    data = np.asarray(t.data if hasattr(t, "data") else t, dtype=np.float64)
    if data.ndim != 3:
        raise ShapeError(f"expected [token][head][dim], got ndim={data.ndim}")
    return torch.from_numpy(np.require(data, None, ["C", "W"])).to(_dev.require_cuda())


def rfft_seq(t) -> ComplexSpectrum:
    """Real FFT along the token axis of every (head, dim) lane (ct/spectral.py:27-34)."""
    x = _seq_device(t)
    spec = torch.fft.rfft(x, dim=0).cpu().numpy()
    return ComplexSpectrum.from_complex(spec, origin_len=int(x.shape[0]))


def lowpass(s: ComplexSpectrum, alpha: float) -> ComplexSpectrum:
    """Zero every bin at index >= floor(alpha * n_freqs) (ct/spectral.py:37-44)."""
    _check_alpha(alpha)
    c = cutoff_index(alpha, s.n_freqs)
    kept = s.to_complex()
    kept[c:] = 0.0
    return ComplexSpectrum.from_complex(kept, origin_len=s.origin_len)


def highpass(s: ComplexSpectrum, alpha: float) -> ComplexSpectrum:
    """Zero the bins below the same cutoff (ct/spectral.py:47-54)."""
    _check_alpha(alpha)
    c = cutoff_index(alpha, s.n_freqs)
    kept = s.to_complex()
    kept[:c] = 0.0
    return ComplexSpectrum.from_complex(kept, origin_len=s.origin_len)


def irfft_seq(s: ComplexSpectrum, n: int) -> SeqTensor:
    """Inverse of rfft_seq back to n real tokens, f32 (ct/spectral.py:61-66)."""
    if n != s.origin_len:
        raise ShapeError(f"requested length {n} != origin_len {s.origin_len}")
    spec = torch.from_numpy(np.require(s.to_complex(), None, ["C", "W"])).to(_dev.require_cuda())
    real = torch.fft.irfft(spec, n=n, dim=0).cpu().numpy()
    return SeqTensor(real.astype(np.float32))


def jaccard_overlap(a, b) -> float:
    """|a & b| / |a | b| of two index sets; 1.0 when both are empty (ct/spectral.py:187-193)."""
    a = np.unique(np.asarray(a, dtype=np.int64))
    b = np.unique(np.asarray(b, dtype=np.int64))
    union = np.union1d(a, b).size
    if union == 0:
        return 1.0
    return np.intersect1d(a, b, assume_unique=True).size / union


def selection_stability(chunk, alphas=(0.3, 0.5, 0.7), r: float = 0.15) -> dict:
    """Jaccard overlap of the top-r selections across cutoff ratios
    (ct/spectral.py:196-208); every ranking runs on the device scorer."""
    picks = {a: indices_for_ratio(rank_chunk(chunk, a), r) for a in alphas}
    out = {}
    for i, a in enumerate(alphas):
        for b in alphas[i + 1:]:
            out[(a, b)] = jaccard_overlap(picks[a], picks[b])
    return out
