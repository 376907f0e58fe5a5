"""ctypes binding of libcachetune_b200.so (include/cachetune_b200.h).

The extension is mandatory: importing the package does not require it, but the
first kernel call raises `NativeLibraryMissing` if the in-tree .so cannot be
loaded -- there is no CPU or eager-PyTorch fallback for any hot-path op.
Statuses map onto the reference exception classes (ct/errors.py:4-37).
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

from .errors import (CacheTuneError, InvalidParam, InvalidPlan, IoError,
                     ShapeError)

LIB_PATH = Path(__file__).resolve().parent / "libcachetune_b200.so"

CT_F32, CT_BF16, CT_F64 = 0, 1, 2
CT_ROPE_ADJACENT, CT_ROPE_SPLIT = 0, 1
CT_MAX_SEGMENTS = 64


class NativeLibraryMissing(CacheTuneError, RuntimeError):
    """libcachetune_b200.so is not built / not loadable (no fallback exists)."""


class CudaError(CacheTuneError, RuntimeError):
    """A CUDA runtime call inside the extension failed."""


class Unsupported(CacheTuneError, NotImplementedError):
    """Geometry not handled by this build."""


_STATUS = {1: ShapeError, 2: InvalidParam, 3: InvalidPlan, 4: IoError,
           5: CudaError, 6: Unsupported}

c_void_p, c_int, c_int64, c_double, c_size_t = (ctypes.c_void_p, ctypes.c_int,
                                                ctypes.c_int64, ctypes.c_double,
                                                ctypes.c_size_t)


class Segment(ctypes.Structure):
    """ct_segment (include/cachetune_b200.h)."""
    _fields_ = [("k", c_void_p), ("v", c_void_p), ("tok", c_void_p),
                ("rows", c_int64), ("pos0", c_int64), ("src_by_tok", c_int64)]


# name -> (restype, argtypes)
_SIGS = {
    "ct_version": (c_int, []),
    "ct_last_error": (c_int, [ctypes.c_char_p, c_size_t]),
    "ct_device_sm_count": (c_int, []),
    "ct_launch_stats": (c_int, [ctypes.c_char_p, c_size_t]),
    "ct_launch_stats_reset": (None, []),
    "ct_score_workspace_bytes": (c_size_t, [c_int64, c_int64, c_int64, c_int64, c_int]),
    "ct_score_chunks": (c_int, [c_void_p, c_void_p, c_int, c_int64, c_int64, c_int64, c_int64,
                                c_int64, c_int64, c_int64, c_int64, c_int, c_void_p, c_void_p,
                                c_void_p, c_void_p, c_void_p, c_size_t, c_void_p]),
    "ct_score_chunks_band": (c_int, [c_void_p, c_void_p, c_int, c_int64, c_int64, c_int64,
                                     c_int64, c_int64, c_int64, c_int64, c_int64, c_int, c_int,
                                     c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_size_t,
                                     c_void_p]),
    "ct_desc_order": (c_int, [c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "ct_score_fast_workspace_bytes": (c_size_t, [c_int64, c_int64, c_int64, c_int64]),
    "ct_score_select_fast": (c_int, [c_void_p, c_void_p, c_int, c_int64, c_int64, c_int64,
                                     c_int64, c_int64, c_int64, c_int64, c_int64, c_int,
                                     c_int64, c_double, c_void_p, c_void_p, c_void_p, c_void_p,
                                     c_void_p, c_size_t, c_void_p]),
    "ct_score_chunk": (c_int, [c_void_p, c_void_p, c_int, c_int64, c_int64, c_int64, c_int64,
                               c_int64, c_double, c_void_p, c_void_p, c_void_p, c_void_p,
                               c_size_t, c_void_p]),
    "ct_select": (c_int, [c_void_p, c_int64, c_double, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ct_selection_plan": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64,
                                  c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "ct_rope_table": (c_int, [c_void_p, c_int64, c_int64, c_double, c_void_p, c_void_p,
                              c_void_p, c_void_p]),
    "ct_rope_apply": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_int, c_int,
                              c_void_p, c_void_p, c_void_p]),
    "ct_gather_rope_blend": (c_int, [ctypes.POINTER(Segment), c_int, c_int64, c_int64,
                                     c_int64, c_int, c_int, c_void_p, c_void_p, c_void_p,
                                     c_int64, c_void_p]),
    "ct_qkv_rope_scatter": (c_int, [c_void_p, c_int64, c_int, c_void_p, c_int64, c_int64,
                                    c_int64, c_int64, c_int, c_void_p, c_void_p, c_int,
                                    c_void_p, c_void_p, c_int, c_int64, c_void_p, c_void_p]),
    "ct_scatter_rows": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "ct_gather_rows": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p]),
    "ct_pool_permute": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int64, c_int64,
                                c_int64, c_int64, c_void_p, c_void_p, c_void_p]),
    "ct_attention_workspace_bytes": (c_size_t, [c_int64, c_int64, c_int64, c_int64, c_int64,
                                                c_int]),
    "ct_selective_attention": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p,
                                       c_void_p, c_int64, c_int64, c_int64, c_int64, c_double,
                                       c_int, c_void_p, c_int, c_void_p, c_void_p, c_size_t,
                                       c_void_p]),
    "ct_embedding_gather": (c_int, [c_void_p, c_void_p, c_int64, c_int64, c_void_p,
                                    c_void_p]),
    "ct_residual_rmsnorm": (c_int, [c_void_p, c_void_p, c_int, c_int64, c_int64, c_double,
                                    c_void_p, c_int, c_void_p]),
    "ct_mlp_act": (c_int, [c_void_p, c_int64, c_int64, c_int, c_int, c_void_p, c_int,
                           c_void_p]),
    "ct_gemm_swiglu": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_int64,
                               c_void_p, c_int64, c_void_p]),
    "ct_gemm_bf16": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_int64,
                             c_void_p, c_int64, c_int, c_int, c_void_p]),
    "ct_gemm_qkv_rope": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64,
                                 c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p,
                                 c_void_p, c_void_p, c_int64, c_void_p]),
    "ct_copy_ranges_h2d": (c_int, [c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
    "ct_host_alloc": (c_int, [ctypes.POINTER(c_void_p), c_size_t]),
    "ct_host_free": (c_int, [c_void_p]),
}

EXPORTS = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


def load(path: Path | str | None = None):
    """Load (once) and return the ctypes library object."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise NativeLibraryMissing(
                f"{p} is missing: run `python -m paper_2605_24022_b200._build` "
                "(there is no CPU fallback)")
        try:
            lib = ctypes.CDLL(str(p))
        except OSError as e:
            raise NativeLibraryMissing(f"cannot load {p}: {e}") from e
        for name, (res, args) in _SIGS.items():
            try:
                fn = getattr(lib, name)
            except AttributeError:
                if path is None:  # the in-tree library must export everything
                    raise
                continue          # an older build loaded for an A/B comparison
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def last_error() -> str:
    buf = ctypes.create_string_buffer(512)
    load().ct_last_error(buf, 512)
    return buf.value.decode(errors="replace")


def launch_stats() -> dict:
    """Kernel name -> successful launches since load / the last reset, as
    counted inside the .so (ct_launch_stats)."""
    buf = ctypes.create_string_buffer(8192)
    check(load().ct_launch_stats(buf, 8192), "ct_launch_stats")
    out = {}
    for item in buf.value.decode().split(";"):
        if item:
            name, _, n = item.rpartition("=")
            out[name] = int(n)
    return out


def launch_stats_reset() -> None:
    load().ct_launch_stats_reset()


# kernel-launching entry points seen through check()/call() (bench evidence)
LAUNCH_COUNT = {"n": 0}
_NOT_KERNELS = {"ct_copy_ranges_h2d", "ct_host_alloc", "ct_host_free", "ct_launch_stats"}


_DEBUG_SYNC = bool(int(__import__("os").environ.get("CT_DEBUG_SYNC", "0")))


def check(status: int, what: str = "") -> None:
    if what not in _NOT_KERNELS:
        LAUNCH_COUNT["n"] += 1
    if _DEBUG_SYNC and status == 0:
        import torch
        try:
            torch.cuda.synchronize()
        except Exception as e:  # attribute the failure to this entry point
            raise CudaError(f"{what}: {e}") from e
    if status != 0:
        cls = _STATUS.get(status, CacheTuneError)
        raise cls(f"{what}: {last_error()}" if what else last_error())


def call(name: str, *args) -> None:
    """Call an int-status entry point and raise the mapped exception."""
    check(getattr(load(), name)(*args), name)
