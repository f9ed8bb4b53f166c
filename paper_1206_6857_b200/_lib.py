"""ctypes binding of the C ABI in include/fastgauss_b200.h.

The engine lives in ``libfastgauss_b200.so`` next to this file (built
in-tree by ``make -C paper_1206_6857_b200/csrc`` or
``python -c "import __graft_entry__ as g; g.build()"``).  There is no CPU
fallback: if the library is missing or a CUDA call fails, the Python API
raises.
"""

from __future__ import annotations

import contextlib
import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FG_LIB selects an alternative in-tree build (engine variants for experiments)
LIB_PATH = os.environ.get("FG_LIB") or os.path.join(_HERE, "libfastgauss_b200.so")

FG_OK, FG_EINVAL, FG_ESTALE, FG_ECUDA, FG_EUNSUPPORTED = 0, 1, 2, 3, 4
MODES = {"dfd": 1, "dfdo": 2, "dito": 3}

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_F64 = ctypes.c_double


class fg_counters(ctypes.Structure):
    _fields_ = [("pair_visits", _I64), ("base_cases", _I64), ("fd_prunes", _I64),
                ("hermite_prunes", _I64), ("local_prunes", _I64), ("h2l_prunes", _I64),
                ("exact_pairs", _I64), ("fp32_pairs", _I64), ("hermite_evals", _I64),
                ("hermite_terms", _I64), ("local_evals", _I64)]


# name -> argtypes (all functions return int status except fg_last_error)
SIGNATURES = {
    "fg_version": [],
    "fg_last_error": [],
    "fg_set_stream": [_P],
    "fg_get_stream": [ctypes.POINTER(_P)],
    "fg_set_device": [ctypes.c_int],
    "fg_synchronize": [],
    "fg_naive_sum": [_P, _I64, _P, _P, _I64, _I32, _P, _I32, _P],
    "fg_tree_build": [_P, _P, _I64, _I32, _I32, ctypes.POINTER(_P)],
    "fg_tree_free": [_P],
    "fg_tree_info": [_P, _P, _P, _P, _P, _P],
    "fg_tree_export": [_P] * 11,
    "fg_tree_points": [_P, _P, _P],
    "fg_moments_refresh": [_P, _F64, _I32],
    "fg_moments_export": [_P, _P, _P, _P, _P],
    "fg_run": [_P, _P, _F64, _F64, _I32, _I32, _P, _P, _P],
    "fg_engine_plimit": [_I32],
    "fg_query_blocks": [_P, _P],
    "fg_query_block_ranges": [_P, _P, _P],
    "fg_run_audit": [_P, _P, _F64, _F64, _I32, _I32, _P, _P, _P, _P, _I64, _P],
    "fg_run_range": [_P, _P, _F64, _F64, _I32, _I32, _I64, _I64, _I64, _P, _P, _P],
    "fg_run_sweep": [_P, _P, _P, _I32, _F64, _I32, _I32, _P, _P, _P],
    "fg_run_sweep_range": [_P, _P, _P, _I32, _F64, _I32, _I32, _I64, _I64, _I64, _P, _P, _P],
    "fg_launch_count": [_P],
    "fg_fp64_peak": [_P],
    "fg_ex2_peak": [_P],
    "fg_set_engine_params": [_I32, _I32, _I32],
    "fg_series_accumulate": [_I32, _P, _P, _P, _I32, _I32, _P, _I32, _F64, _P],
    "fg_series_eval": [_I32, _P, _I32, _P, _I32, _I32, _I32, _F64, _P, _P, _P],
    "fg_series_translate": [_I32, _P, _I32, _P, _P, _I32, _I32, _I32, _I32, _F64, _P],
    "fg_best_method": [_P, _I32, _I32, _I32, _P],
    "fg_iset_export": [_I32, _I32, _P, _P, _P, _P, _P, _P, _P],
    "fg_check_failures": [_P],
}

_lib = None
_lock = threading.Lock()


class EngineMissing(RuntimeError):
    pass


def lib():
    """Load the engine library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise EngineMissing(
                    f"{LIB_PATH} is missing: build it with `make -C "
                    f"{os.path.join(_HERE, 'csrc')}` (there is no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            for name, args in SIGNATURES.items():
                fn = getattr(L, name)
                fn.argtypes = args
                fn.restype = ctypes.c_char_p if name == "fg_last_error" else ctypes.c_int
            _lib = L
    return _lib


def check(status: int, what: str = "") -> None:
    if status == FG_OK:
        return
    msg = lib().fg_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if status in (FG_EINVAL, FG_EUNSUPPORTED):
        raise ValueError(msg)
    if status == FG_ESTALE:
        raise RuntimeError(msg)
    raise RuntimeError(f"CUDA error: {msg}")


def call(name: str, *args):
    check(getattr(lib(), name)(*args), name)


# --------------------------------------------------------------- buffers
def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def ptr(x):
    """Raw pointer of a numpy array or a torch tensor (host or CUDA)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    if _is_torch(x):
        return x.data_ptr()
    raise TypeError(f"unsupported buffer type {type(x)!r}")


def as_f64(x, ndim=None):
    """Contiguous float64 view of array-like input (torch tensors kept as-is)."""
    if _is_torch(x):
        import torch

        t = x.to(torch.float64).contiguous()
        return t
    a = np.ascontiguousarray(x, dtype=np.float64)
    if ndim is not None and a.ndim != ndim:
        raise ValueError(f"expected a {ndim}-d array")
    return a


def set_stream(stream_handle: int | None) -> None:
    """Set the calling thread's engine stream (None: per-thread default)."""
    call("fg_set_stream", stream_handle)


def get_stream() -> int | None:
    s = ctypes.c_void_p()
    call("fg_get_stream", ctypes.byref(s))
    return s.value


@contextlib.contextmanager
def torch_stream(*objs):
    """Run the engine on torch's current stream while any of ``objs`` is a
    CUDA tensor, so the call is ordered after the torch work that produced
    (or zeroed) those tensors; the thread's previous engine stream is restored
    afterwards."""
    t = next((o for o in objs if _is_torch(o) and o.is_cuda), None)
    if t is None:
        yield
        return
    import torch

    cur = torch.cuda.current_stream(t.device).cuda_stream or None
    prev = get_stream()
    if cur == prev:
        yield
        return
    set_stream(cur)
    try:
        yield
    finally:
        set_stream(prev)


def check_out(out, shapes, what: str = "out"):
    """Validate a caller-supplied output buffer before its raw pointer reaches
    the C ABI: float64, C-contiguous, writeable, one of ``shapes``; a CUDA
    tensor must be on the current device.  Raises ValueError."""
    if out is None:
        return None
    shapes = [tuple(int(d) for d in sh) for sh in shapes]
    if isinstance(out, np.ndarray):
        ok = (out.dtype == np.float64 and out.flags.c_contiguous and out.flags.writeable
              and tuple(out.shape) in shapes)
        if not ok:
            raise ValueError(f"{what} must be a writeable C-contiguous float64 array of shape "
                             f"{' or '.join(map(str, shapes))}; got {out.dtype} {out.shape}")
        return out
    if _is_torch(out):
        import torch

        ok = (out.dtype == torch.float64 and out.is_contiguous()
              and tuple(out.shape) in shapes)
        if not ok:
            raise ValueError(f"{what} must be a contiguous float64 tensor of shape "
                             f"{' or '.join(map(str, shapes))}; got {out.dtype} "
                             f"{tuple(out.shape)}")
        if out.is_cuda and out.device.index != torch.cuda.current_device():
            raise ValueError(f"{what} is on {out.device}, the engine runs on "
                             f"cuda:{torch.cuda.current_device()}")
        return out
    raise ValueError(f"{what} must be a NumPy array or a torch tensor")
