"""ctypes wrapper over oracle/_build/librtk_oracle.so -- TEST INFRASTRUCTURE ONLY.

Each wrapper mirrors the reference function it restates:
  exact_topk   -> _kernels.exact_topk_chunk  (_kernels.py:165-186)
  early_topk   -> _kernels.early_topk_chunk  (_kernels.py:189-214)
  exact_trace  -> _kernels.exact_trace_chunk (_kernels.py:217-231)
  row_min_max  -> _kernels.row_min_max       (_kernels.py:26-36)
  count_ge     -> _kernels.count_ge          (_kernels.py:39-45)
  first_nan_row-> batch.as_matrix NaN scan   (batch.py:37-39)
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

EXIT_COUNT_EQUALS_K = 1
EXIT_INTERVAL_BELOW_EPSILON = 2
EXIT_MAX_ITER_REACHED = 3
EXIT_HARD_CAP_REACHED = 4
EXIT_DEGENERATE_ROW = 5

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "librtk_oracle.so")
_lock = threading.Lock()
_lib = None

_f32p = ctypes.POINTER(ctypes.c_float)
_i32p = ctypes.POINTER(ctypes.c_int32)
_i8p = ctypes.POINTER(ctypes.c_int8)
_i64 = ctypes.c_int64


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (gcc only)."""
    src = os.path.join(_HERE, "rtk_oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_SO):
                build()
            L = ctypes.CDLL(_SO)
            L.rtko_exact_topk.argtypes = [_f32p, _i64, _i64, _i64, ctypes.c_int32, ctypes.c_double,
                                          ctypes.c_int32, _f32p, _i32p, _i64, _i32p, _i8p, ctypes.c_int]
            L.rtko_exact_topk.restype = None
            L.rtko_early_topk.argtypes = [_f32p, _i64, _i64, _i64, ctypes.c_int32, ctypes.c_int32,
                                          _f32p, _i32p, _i64, _i32p, _i8p, ctypes.c_int]
            L.rtko_early_topk.restype = None
            L.rtko_exact_trace.argtypes = [_f32p, _i64, _i64, _i64, ctypes.c_int32, ctypes.c_double,
                                           ctypes.c_int32, _i32p, _i8p, ctypes.c_int]
            L.rtko_exact_trace.restype = None
            L.rtko_first_nan_row.argtypes = [_f32p, _i64, _i64, _i64]
            L.rtko_first_nan_row.restype = _i64
            L.rtko_row_min_max.argtypes = [_f32p, _i64, _f32p, _f32p]
            L.rtko_row_min_max.restype = None
            L.rtko_count_ge.argtypes = [_f32p, _i64, ctypes.c_float]
            L.rtko_count_ge.restype = _i64
            L.rtko_mid_f32.argtypes = [ctypes.c_float, ctypes.c_float]
            L.rtko_mid_f32.restype = ctypes.c_float
            L.rtko_mid_f64.argtypes = [ctypes.c_float, ctypes.c_float]
            L.rtko_mid_f64.restype = ctypes.c_float
            L.rtko_mid_mismatches.argtypes = [ctypes.c_void_p, ctypes.c_void_p, _i64]
            L.rtko_mid_mismatches.restype = _i64
            L.rtko_max_threads.argtypes = []
            L.rtko_max_threads.restype = ctypes.c_int
            _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


def _matrix(x) -> np.ndarray:
    m = np.ascontiguousarray(x, dtype=np.float32)
    if m.ndim != 2:
        raise ValueError(f"expected 2-D, got {m.shape}")
    return m


def exact_topk(x, k: int, eps_rel: float = 0.0, hard_cap: int = 64, threads: int = 0):
    m = _matrix(x)
    n, cols = m.shape
    vals = np.empty((n, k), np.float32)
    idx = np.empty((n, k), np.int32)
    iters = np.zeros(n, np.int32)
    reasons = np.zeros(n, np.int8)
    lib().rtko_exact_topk(_p(m, _f32p), n, cols, cols, int(k), float(eps_rel), int(hard_cap),
                          _p(vals, _f32p), _p(idx, _i32p), k, _p(iters, _i32p), _p(reasons, _i8p),
                          int(threads))
    return vals, idx, iters, reasons


def early_topk(x, k: int, max_iter: int = 4, threads: int = 0):
    m = _matrix(x)
    n, cols = m.shape
    vals = np.empty((n, k), np.float32)
    idx = np.empty((n, k), np.int32)
    iters = np.zeros(n, np.int32)
    reasons = np.zeros(n, np.int8)
    lib().rtko_early_topk(_p(m, _f32p), n, cols, cols, int(k), int(max_iter),
                          _p(vals, _f32p), _p(idx, _i32p), k, _p(iters, _i32p), _p(reasons, _i8p),
                          int(threads))
    return vals, idx, iters, reasons


def exact_trace(x, k: int, eps_rel: float = 0.0, hard_cap: int = 64, threads: int = 0):
    m = _matrix(x)
    n, cols = m.shape
    iters = np.zeros(n, np.int32)
    reasons = np.zeros(n, np.int8)
    lib().rtko_exact_trace(_p(m, _f32p), n, cols, cols, int(k), float(eps_rel), int(hard_cap),
                           _p(iters, _i32p), _p(reasons, _i8p), int(threads))
    return iters, reasons


def ref_batch(x, k: int, mode: str = "exact", max_iter: int = 4, eps_rel: float = 0.0,
              hard_cap: int = 64, threads: int = 0):
    """(values, indices, trace_iterations, trace_reasons) exactly as the reference's
    batch_topk(x, BatchConfig(k, search, collect_traces=True)) returns them."""
    if mode == "exact":
        return exact_topk(x, k, eps_rel, hard_cap, threads)
    if mode in ("early", "early-stop", "early_stop"):
        return early_topk(x, k, max_iter, threads)
    raise ValueError(mode)


def first_nan_row(x) -> int:
    m = _matrix(x)
    return int(lib().rtko_first_nan_row(_p(m, _f32p), m.shape[0], m.shape[1], m.shape[1]))


def row_min_max(v):
    v = np.ascontiguousarray(v, dtype=np.float32)
    mn = ctypes.c_float()
    mx = ctypes.c_float()
    lib().rtko_row_min_max(_p(v, _f32p), v.shape[0], ctypes.byref(mn), ctypes.byref(mx))
    return np.float32(mn.value), np.float32(mx.value)


def count_ge(v, t) -> int:
    v = np.ascontiguousarray(v, dtype=np.float32)
    return int(lib().rtko_count_ge(_p(v, _f32p), v.shape[0], float(np.float32(t))))


def mid_f32(a, b) -> np.float32:
    return np.float32(lib().rtko_mid_f32(float(np.float32(a)), float(np.float32(b))))


def mid_f64(a, b) -> np.float32:
    return np.float32(lib().rtko_mid_f64(float(np.float32(a)), float(np.float32(b))))


def max_threads() -> int:
    return int(lib().rtko_max_threads())


def mid_mismatches(a_bits, b_bits) -> int:
    a = np.ascontiguousarray(a_bits, np.uint32)
    b = np.ascontiguousarray(b_bits, np.uint32)
    return int(lib().rtko_mid_mismatches(a.ctypes.data, b.ctypes.data, a.size))
