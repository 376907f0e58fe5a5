"""(3) Deferred RoPE at true global positions (drop-in for ct/rope.py).

`RopeParams` validates exactly like ct/rope.py:20-44.  The (cos, sin) table is
built on the device in float64 from the host-computed frequencies
base**(-2j/D) (numpy, the reference's own expression) and cached per
(params, device); kernels read it from L2.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _dev, _lib
from .errors import InvalidParam, ShapeError
from .kvcore import SeqTensor


@dataclass(frozen=True)
class RopeParams:
    head_dim: int
    base: float = 10000.0
    scaling: float = 1.0
    pairing: str = "adjacent"

    def __post_init__(self):
        if self.base <= 1.0:
            raise InvalidParam(f"base must be > 1, got {self.base}")
        if self.head_dim < 2 or self.head_dim % 2 != 0:
            raise InvalidParam(f"head_dim must be even and >= 2, got {self.head_dim}")
        if self.pairing not in ("adjacent", "split"):
            raise InvalidParam(f"unknown pairing {self.pairing!r}")

    def freqs(self) -> np.ndarray:
        """base ** (-2 j / D) in float64 (ct/rope.py:42-44)."""
        j = np.arange(self.head_dim // 2, dtype=np.float64)
        return self.base ** (-2.0 * j / self.head_dim)

    @property
    def pairing_code(self) -> int:
        return _lib.CT_ROPE_ADJACENT if self.pairing == "adjacent" else _lib.CT_ROPE_SPLIT


def as_rope_params(p) -> RopeParams:
    if isinstance(p, RopeParams):
        return p
    return RopeParams(int(p.head_dim), float(p.base), float(p.scaling), str(p.pairing))


_tables: dict = {}
_tables_lock = threading.Lock()


def rope_table(params: RopeParams, n_pos: int, kind: str, device) -> torch.Tensor:
    """(cos, sin) table [n_pos_cap, D/2, 2] in f64 ("f64") or f32 ("f32")."""
    params = as_rope_params(params)
    device = torch.device(device)
    key = (params, kind, device)
    with _tables_lock:
        t = _tables.get(key)
        if t is not None and t.shape[0] >= n_pos:
            return t
        cap = 1 << max(10, int(np.ceil(np.log2(max(n_pos, 1)))))
        half = params.head_dim // 2
        freqs = torch.as_tensor(params.freqs(), device=device)
        dt = torch.float64 if kind == "f64" else torch.float32
        t = torch.empty((cap, half, 2), dtype=dt, device=device)
        _lib.call("ct_rope_table", _dev.ptr(freqs), half, cap, float(params.scaling), None,
                  _dev.ptr(t) if kind == "f64" else None,
                  _dev.ptr(t) if kind == "f32" else None, _dev.stream_handle())
        _tables[key] = t
        return t


def rope_table_for(params: RopeParams, positions: torch.Tensor, kind: str) -> torch.Tensor:
    """Per-row table for an arbitrary (possibly negative) int64 position list."""
    params = as_rope_params(params)
    half = params.head_dim // 2
    freqs = torch.as_tensor(params.freqs(), device=positions.device)
    dt = torch.float64 if kind == "f64" else torch.float32
    t = torch.empty((positions.numel(), half, 2), dtype=dt, device=positions.device)
    pos = positions.to(torch.int64).contiguous()
    _lib.call("ct_rope_table", _dev.ptr(freqs), half, pos.numel(), float(params.scaling),
              _dev.ptr(pos), _dev.ptr(t) if kind == "f64" else None,
              _dev.ptr(t) if kind == "f32" else None, _dev.stream_handle())
    return t


def rope_apply_device(x: torch.Tensor, positions: torch.Tensor, params) -> torch.Tensor:
    """Rotate [n, H, D] rows at device positions (f32 rows rotate in f64 math)."""
    params = as_rope_params(params)
    n, h, d = x.shape
    if d != params.head_dim:
        raise ShapeError(f"tensor head_dim {d} != params head_dim {params.head_dim}")
    if positions.numel() != n:
        raise ShapeError(f"{positions.numel()} positions for {n} tokens")
    x = x.contiguous()
    out = torch.empty_like(x)
    if n == 0:
        return out
    kind = "f64" if x.dtype in (torch.float32, torch.float64) else "f32"
    tab = rope_table_for(params, positions, kind)
    rows = torch.arange(n, dtype=torch.int32, device=x.device)
    _lib.call("ct_rope_apply", _dev.ptr(x), _dev.ptr(rows), n, h, d,
              _dev.ct_dtype(x.dtype), params.pairing_code, _dev.ptr(tab), _dev.ptr(out),
              _dev.stream_handle())
    return out


def rope_apply(keys, positions: Sequence[int], params) -> SeqTensor:
    """Apply the rotary transform to each token's key at its position (ct/rope.py:75-81)."""
    params = as_rope_params(params)
    data = np.asarray(keys.data if hasattr(keys, "data") else keys, dtype=np.float32)
    pos = np.asarray(positions)
    if pos.shape != (data.shape[0],):
        raise ShapeError(f"{pos.size} positions for {data.shape[0]} tokens")
    if data.shape[2] != params.head_dim:
        raise ShapeError(f"tensor head_dim {data.shape[2]} != params head_dim {params.head_dim}")
    dev = _dev.require_cuda()
    x = torch.from_numpy(np.require(data, None, ["C", "W"])).to(dev)
    p = torch.as_tensor(pos.astype(np.int64), device=dev)
    return SeqTensor(rope_apply_device(x, p, params).cpu().numpy())


def rope_rotate(x, positions, params):
    """ct/rope.py:47-72: rotate an [N, H, D] array at `positions` in float64
    arithmetic and return float64 (numpy in -> numpy out, torch -> torch on
    the device).  ct_rope_apply with f64 rows: unfused products and sums, so
    the result equals numpy's up to the cos/sin of the angle table (<= 1 ulp)."""
    params = as_rope_params(params)
    as_numpy = not isinstance(x, torch.Tensor)
    shape = tuple(np.shape(x))
    if len(shape) != 3:
        raise ShapeError(f"expected [N, H, D], got shape {shape}")
    if shape[2] != params.head_dim:
        raise ShapeError(f"tensor head_dim {shape[2]} != params head_dim {params.head_dim}")
    dev = _dev.require_cuda() if as_numpy else x.device
    xt = (torch.from_numpy(np.require(x, np.float64, ["C", "W"])).to(dev) if as_numpy
          else x.to(torch.float64))
    pos = torch.as_tensor(np.asarray(positions, dtype=np.int64) if as_numpy
                          else positions, device=dev).to(torch.int64)
    if pos.numel() != shape[0]:
        raise ShapeError(f"{pos.numel()} positions for {shape[0]} tokens")
    out = rope_apply_device(xt, pos, params)
    return out.cpu().numpy() if as_numpy else out
