"""ctypes binding of librtk.so (the C ABI in include/rtk.h).

This is the only way the package computes: there is no CPU fallback.  A
missing library or a missing CUDA device raises DeviceError.
"""

from __future__ import annotations

import ctypes
import os
import threading

from ._build import SO
from .errors import DeviceError

RTK_OK, RTK_EINVAL, RTK_ECUDA, RTK_EIO, RTK_EFORMAT, RTK_ETRUNC, RTK_ENAN, RTK_EUNSUPPORTED = 0, 1, 2, 3, 4, 5, 6, 7

_lock = threading.Lock()
_lib = None

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32

# name -> (restype, argtypes); must match include/rtk.h exactly
SIGNATURES = {
    "rtk_rowtopk_exact_f32": (ctypes.c_int, [_p, _i64, _i64, _i64, _i32, ctypes.c_double, _i32,
                                             _p, _p, _i64, _p, _p, _p, _p]),
    "rtk_rowtopk_early_f32": (ctypes.c_int, [_p, _i64, _i64, _i64, _i32, _i32,
                                             _p, _p, _i64, _p, _p, _p, _p]),
    "rtk_exact_trace_f32": (ctypes.c_int, [_p, _i64, _i64, _i64, _i32, ctypes.c_double, _i32,
                                           _p, _p, _p, _p]),
    "rtk_rowtopk_x16": (ctypes.c_int, [_p, _i32, _i32, _i64, _i64, _i64, _i32, _i32, _i32, _p, _p, _i64, _p, _p]),
    "rtk_maxk_dense": (ctypes.c_int, [_p, _i32, _i32, _i64, _i64, _i64, _i32, _i32, _i32, _p, _p, _i64, _p, _i64,
                                      _p, _i64, _p, _p]),
    "rtk_nan_scan_f32": (ctypes.c_int, [_p, _i64, _i64, _i64, _p, _p]),
    "rtk_row_min_max_f32": (ctypes.c_int, [_p, _i64, _i64, _i64, _p, _p, _p]),
    "rtk_count_ge_f32": (ctypes.c_int, [_p, _i64, _i64, _i64, _p, _p, _p]),
    "rtk_topk_file_f32": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_char_p, _i32, _i32, ctypes.c_double, _i32, _i32,
                                         _i64, _p]),
    "rtk_scatter_rows_f32": (ctypes.c_int, [_p, _p, _i64, _i64, _i32, _i64, _p, _i64, _p]),
    "rtk_gather_rows_f32": (ctypes.c_int, [_p, _i64, _p, _i64, _i64, _i32, _i64, _p, _p]),
    "rtk_maxk_spmm_f32": (ctypes.c_int, [_p, _p, _p, _i64, _p, _p, _p, _i64, _i32, _i64, _i64, _p, _i64, _p]),
    "rtk_maxk_spmm_backward_f32": (ctypes.c_int, [_p, _p, _p, _i64, _p, _i64, _p, _p, _i64, _i32, _i64, _p, _p]),
    "rtk_last_error": (ctypes.c_char_p, []),
    "rtk_version": (ctypes.c_int, []),
    "rtk_launch_shape": (ctypes.c_int, [_i64, _i32, _i32, _p, _p, _p]),
}


def library_path() -> str:
    return os.environ.get("RTK_LIBRARY", SO)


def load():
    """Load librtk.so once (raises DeviceError when it is not built)."""
    global _lib
    with _lock:
        if _lib is None:
            path = library_path()
            if not os.path.exists(path):
                raise DeviceError(f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                                  " (there is no CPU fallback)")
            lib = ctypes.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    if rc != RTK_OK:
        msg = load().rtk_last_error().decode(errors="replace")
        raise DeviceError(f"{what} failed (rc={rc}): {msg}")


def last_error() -> str:
    return load().rtk_last_error().decode(errors="replace")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
