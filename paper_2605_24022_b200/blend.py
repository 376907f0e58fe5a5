"""(2)+(3) Scatter fusion of reused (deferred-RoPE) and recomputed KV.

Drop-in for ct/pipesim.py:322-357 (fuse_layer) and ct/kvcore.py:171-194
(tensor_scatter_tokens).  Validation is host-side and identical to the
reference (InvalidPlan on a non-partition, ShapeError on geometry); the row
movement and rotation run in the fused ct_gather_rope_blend kernel.
"""

from __future__ import annotations

from typing import Sequence

import numpy as np
import torch

from . import _dev, _lib
from .errors import InvalidPlan, ShapeError
from .kvcore import SeqTensor, check_scatter
from .rope import as_rope_params, rope_apply_device, rope_table


def _to_dev(t, dev):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return t.to(dev).contiguous()
    data = t.data if hasattr(t, "data") and not isinstance(t, np.ndarray) else t
    return torch.from_numpy(np.require(data, np.float32, ["C", "W"])).to(dev)


def scatter_rows_device(dst: torch.Tensor, src: torch.Tensor, idx: torch.Tensor) -> None:
    """dst[idx[i]] = src[i] for [rows, ...] tensors (ct/kvcore.py:192-193)."""
    n = idx.numel()
    if n == 0:
        return
    row_bytes = src[0].numel() * src.element_size()
    _lib.call("ct_scatter_rows", _dev.ptr(src.contiguous()), _dev.ptr(idx.to(torch.int32)),
              n, row_bytes, _dev.ptr(dst), _dev.stream_handle())


def gather_rows_device(src: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
    """out[i] = src[idx[i]]."""
    n = idx.numel()
    out = torch.empty((n, *src.shape[1:]), dtype=src.dtype, device=src.device)
    if n:
        row_bytes = src[0].numel() * src.element_size()
        _lib.call("ct_gather_rows", _dev.ptr(src.contiguous()), _dev.ptr(idx.to(torch.int32)),
                  n, row_bytes, _dev.ptr(out), _dev.stream_handle())
    return out


def fuse_layer_device(k_reuse, v_reuse, keep: np.ndarray, k_new, v_new, rec: np.ndarray,
                      positions: np.ndarray, rope_params, n: int, dev):
    params = as_rope_params(rope_params)
    ref = k_reuse if k_reuse is not None else k_new
    h, d = ref.shape[1], ref.shape[2]
    kbuf = torch.empty((n, h, d), dtype=ref.dtype, device=dev)
    vbuf = torch.empty_like(kbuf)
    if keep.size:
        keep_d = torch.as_tensor(keep.astype(np.int32), device=dev)
        if np.array_equal(np.asarray(positions), keep) and keep.max() < 2 ** 31:
            # fused gather + deferred RoPE + blend: row i -> keep[i] rotated at keep[i]
            kind = "f64" if ref.dtype == torch.float32 else "f32"
            tab = rope_table(params, int(keep.max()) + 1, kind, dev)
            seg = _lib.Segment(_dev.ptr(k_reuse), _dev.ptr(v_reuse), _dev.ptr(keep_d),
                               keep.size, 0, 0)
            _lib.call("ct_gather_rope_blend", seg, 1, h * d, h, d, _dev.ct_dtype(ref.dtype),
                      params.pairing_code, _dev.ptr(tab), _dev.ptr(kbuf), _dev.ptr(vbuf), h * d,
                      _dev.stream_handle())
        else:
            pos_d = torch.as_tensor(np.asarray(positions, dtype=np.int64), device=dev)
            scatter_rows_device(kbuf, rope_apply_device(k_reuse, pos_d, params), keep_d)
            scatter_rows_device(vbuf, v_reuse, keep_d)
    if rec.size:
        rec_d = torch.as_tensor(rec.astype(np.int32), device=dev)
        scatter_rows_device(kbuf, k_new, rec_d)
        scatter_rows_device(vbuf, v_new, rec_d)
    return kbuf, vbuf


def fuse_layer(reused, recomputed, positions: Sequence[int], rope_params, n: int):
    """Assemble one layer's complete KV (ct/pipesim.py:322-357).

    reused = (K_raw | None, V | None, keep_idx); recomputed = (K | None, V | None,
    rec_idx); reused keys are rotated to `positions`; the index sets must
    partition [0, n).  Returns (SeqTensor K, SeqTensor V)."""
    k_reuse, v_reuse, keep_idx = reused
    k_new, v_new, rec_idx = recomputed
    keep = np.asarray(keep_idx, dtype=np.int64)
    rec = np.asarray(rec_idx, dtype=np.int64)
    merged = np.concatenate([keep, rec])
    if merged.size != n or not np.array_equal(np.sort(merged), np.arange(n)):
        raise InvalidPlan("keep/recompute sets must partition [0, n)")
    parts = [t for t in (k_reuse, k_new) if t is not None]
    if not parts:
        raise InvalidPlan("fusing two empty parts")
    if keep.size:
        pos = np.asarray(positions)
        if pos.shape != (keep.size,):
            raise ShapeError(f"{pos.size} positions for {keep.size} reused tokens")
    dev = _dev.require_cuda()
    kr, vr = _to_dev(k_reuse, dev), _to_dev(v_reuse, dev)
    kn, vn = _to_dev(k_new, dev), _to_dev(v_new, dev)
    for t, want in ((kr, keep.size), (vr, keep.size), (kn, rec.size), (vn, rec.size)):
        if t is not None and t.shape[0] != want:
            raise ShapeError(f"{t.shape[0]} rows for {want} indices")
    kbuf, vbuf = fuse_layer_device(kr, vr, keep, kn, vn, rec, np.asarray(positions), rope_params,
                                   n, dev)
    return SeqTensor(kbuf.cpu().numpy()), SeqTensor(vbuf.cpu().numpy())


def tensor_scatter_tokens(dst, src, indices: Sequence[int]) -> SeqTensor:
    """dst with rows at `indices` replaced by src rows (ct/kvcore.py:171-194)."""
    idx = np.asarray(indices, dtype=np.int64)
    dst_data = np.asarray(dst.data, dtype=np.float32)
    if idx.size == 0:
        return SeqTensor(dst_data.copy())
    src_data = None if src is None else np.asarray(src.data, dtype=np.float32)
    check_scatter(dst_data.shape[0], None if src_data is None else src_data.shape[0],
                  () if src_data is None else src_data.shape[1:], dst_data.shape[1:], idx)
    dev = _dev.require_cuda()
    out = torch.from_numpy(dst_data.copy()).to(dev)
    scatter_rows_device(out, torch.from_numpy(src_data).to(dev),
                        torch.as_tensor(idx.astype(np.int32), device=dev))
    return SeqTensor(out.cpu().numpy())
