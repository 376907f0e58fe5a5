"""Device plumbing: torch tensors -> C-ABI pointers, streams, workspaces.

PyTorch provides HBM allocation, streams and events only; every compute op on
the hot path is a kernel of libcachetune_b200.so.
"""

from __future__ import annotations

import threading

import numpy as np
import torch

from . import _lib

_ws_lock = threading.Lock()
_workspaces: dict = {}


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise _lib.NativeLibraryMissing(
            "no CUDA device: the B200 path has no CPU fallback")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def stream_handle(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def ct_dtype(t: torch.dtype) -> int:
    if t == torch.float32:
        return _lib.CT_F32
    if t == torch.bfloat16:
        return _lib.CT_BF16
    if t == torch.float64:
        return _lib.CT_F64
    raise _lib.Unsupported(f"dtype {t}")


def workspace(nbytes: int, tag: str = "default") -> torch.Tensor | None:
    """Per-(device, stream, tag) grow-only workspace."""
    if nbytes <= 0:
        return None
    dev = torch.cuda.current_device()
    key = (dev, torch.cuda.current_stream().cuda_stream, tag)
    with _ws_lock:
        buf = _workspaces.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(int(nbytes * 1.25) + 256, dtype=torch.uint8, device=f"cuda:{dev}")
            _workspaces[key] = buf
        return buf


def i32(a, device) -> torch.Tensor:
    return torch.as_tensor(np.asarray(a, dtype=np.int32), device=device)


def i64(a, device) -> torch.Tensor:
    return torch.as_tensor(np.asarray(a, dtype=np.int64), device=device)
