"""CPU-only tests: the C-ABI library loads and exports every declared symbol,
the host-side mirror of the reference API validates like the reference, and
the product path refuses to run without a GPU (no CPU fallback)."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2409_00822_b200 as rtk
from paper_2409_00822_b200 import _build, _native
from paper_2409_00822_b200.shard import shard_range

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "rtk.h")) as f:
        txt = f.read()
    return sorted(set(re.findall(r"RTK_API\s+[\w\s\*]*?\b(rtk_\w+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return _native.load()


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("rtk_rowtopk_exact_f32", "rtk_rowtopk_early_f32", "rtk_exact_trace_f32", "rtk_nan_scan_f32",
              "rtk_last_error"):
        assert s in syms
    assert set(syms) == set(_native.SIGNATURES)


def test_library_loads_and_exports_every_symbol(lib):
    raw = ctypes.CDLL(_native.library_path())
    for s in declared_symbols():
        assert hasattr(raw, s), s
    assert lib.rtk_version() == 100


def test_cabi_rejects_bad_arguments_without_touching_the_gpu(lib):
    # argument checks run before any CUDA call, so they work on a CPU box
    fake = 256  # never dereferenced: every check below fails before a launch
    assert lib.rtk_rowtopk_exact_f32(fake, 4, 8, 8, 9, 0.0, 64, fake, fake, 9, None, None, None, None) == 1
    assert b"k must be in [1, 8], got 9" in lib.rtk_last_error()
    assert lib.rtk_rowtopk_exact_f32(None, 4, 8, 8, 2, 0.0, 64, fake, fake, 2, None, None, None, None) == 1
    assert b"x is NULL" in lib.rtk_last_error()
    assert lib.rtk_rowtopk_early_f32(fake, 4, 8, 8, 2, 0, fake, fake, 2, None, None, None, None) == 1
    assert b"max_iter must be >= 1" in lib.rtk_last_error()
    assert lib.rtk_rowtopk_exact_f32(fake, 4, 8, 8, 2, 0.0, 64, None, fake, 2, None, None, None, None) == 1
    assert b"vals/idx is NULL" in lib.rtk_last_error()
    assert lib.rtk_rowtopk_exact_f32(fake, 4, 8, 4, 2, 0.0, 64, None, None, 2, None, None, None, None) == 1
    assert b"ldx" in lib.rtk_last_error()
    assert lib.rtk_rowtopk_exact_f32(None, -1, 8, 8, 2, 0.0, 64, None, None, 2, None, None, None, None) == 1
    assert lib.rtk_exact_trace_f32(None, 0, 8, 8, 2, -1.0, 64, None, None, None, None) == 1
    assert lib.rtk_launch_shape(8, 9, 0, None, None, None) == 1
    # n == 0 is a no-op
    assert lib.rtk_rowtopk_exact_f32(None, 0, 8, 8, 2, 0.0, 64, None, None, 2, None, None, None, None) == 0
    # fused MaxK rows: dtype, outputs, native-path shape (RTK_EUNSUPPORTED = 7)
    assert lib.rtk_maxk_dense(fake, 3, 0, 4, 256, 256, 8, 64, 4, fake, fake, 8, fake, 256, None, 0, None, None) == 1
    assert b"dtype" in lib.rtk_last_error()
    assert lib.rtk_maxk_dense(fake, 0, 0, 4, 256, 256, 8, 64, 4, fake, fake, 8, None, 0, None, 0, None, None) == 1
    assert b"both NULL" in lib.rtk_last_error()
    assert lib.rtk_maxk_dense(fake, 0, 0, 4, 256, 256, 300, 64, 4, fake, fake, 300, fake, 256, None, 0, None,
                              None) == 1
    assert lib.rtk_maxk_dense(fake, 0, 0, 4, 200, 200, 8, 64, 4, fake, fake, 8, fake, 200, None, 0, None, None) == 7
    assert b"fused MaxK path" in lib.rtk_last_error()
    # aggregation: exactly one index array, width limits, 32-bit offsets
    assert lib.rtk_maxk_spmm_f32(fake, fake, None, 4, fake, fake, fake, 32, 32, 256, 10, fake, 256, None) == 1
    assert b"exactly one of idx / idx8" in lib.rtk_last_error()
    assert lib.rtk_maxk_spmm_f32(fake, fake, None, 4, fake, None, fake, 32, 32, 300, 10, fake, 300, None) == 1
    assert b"m <= 256" in lib.rtk_last_error()
    assert lib.rtk_maxk_spmm_f32(fake, fake, None, 4, fake, fake, None, 32, 32, 2000, 10, fake, 2000, None) == 1
    assert lib.rtk_maxk_spmm_f32(fake, fake, None, 4, fake, fake, None, 32, 32, 256, 1 << 27, fake, 256, None) == 1
    assert b"2^31" in lib.rtk_last_error()
    assert lib.rtk_maxk_spmm_backward_f32(fake, fake, None, 4, fake, 100, fake, None, 32, 32, 256, fake, None) == 1
    assert lib.rtk_maxk_spmm_f32(None, None, None, 0, None, fake, None, 32, 32, 256, 0, None, 256, None) == 0


def test_search_config_validation_mirrors_reference():
    with pytest.raises(ValueError, match="epsilon_rel must be >= 0"):
        rtk.SearchConfig(epsilon_rel=-1.0)
    with pytest.raises(ValueError, match="max_iter must be >= 1"):
        rtk.SearchConfig.early_stop(0)
    with pytest.raises(ValueError, match="hard_cap must be >= 1"):
        rtk.SearchConfig.exact(hard_cap=0)
    assert rtk.SearchConfig().mode is rtk.SearchMode.EXACT
    assert rtk.SearchConfig.early_stop().max_iter == rtk.DEFAULT_MAX_ITER == 4
    assert rtk.SearchConfig.exact().hard_cap == rtk.DEFAULT_HARD_CAP == 64
    assert [int(e) for e in rtk.ExitReason] == [1, 2, 3, 4, 5]


def test_batch_config_and_result_surface():
    cfg = rtk.BatchConfig(k=3)
    assert cfg.workers == "auto" and cfg.collect_traces is False
    assert cfg.search == rtk.SearchConfig.exact()
    res = rtk.BatchResult(np.zeros((2, 3), np.float32), np.zeros((2, 3), np.int32))
    assert res.n_rows == 2 and res.k == 3
    with pytest.raises(ValueError, match="traces were not collected"):
        res.traces()
    tr = rtk.BatchResult(np.zeros((2, 3), np.float32), np.zeros((2, 3), np.int32),
                         np.array([3, 0], np.int32), np.array([1, 5], np.int8)).traces()
    assert tr[0] == rtk.SearchTrace(3, rtk.ExitReason.COUNT_EQUALS_K)
    assert tr[1].exit_reason is rtk.ExitReason.DEGENERATE_ROW


def test_resolve_workers_and_chunk_ranges():
    assert rtk.resolve_workers("auto") >= 1
    assert rtk.resolve_workers(3) == 3
    with pytest.raises(ValueError):
        rtk.resolve_workers(0)
    for n, w in [(1, 1), (10, 3), (100, 8), (7, 16)]:
        covered = [i for a, b in rtk.chunk_ranges(n, w) for i in range(a, b)]
        assert covered == list(range(n))


def test_shard_range_partitions_rows():
    for n in (0, 1, 7, 100, 1 << 20, 232965):
        for world in (1, 2, 3, 4, 8):
            rows = []
            for r in range(world):
                a, b = shard_range(n, r, world)
                rows.extend(range(a, b))
            assert rows == list(range(n))
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    with pytest.raises(rtk.DeviceError, match="no CPU fallback"):
        rtk.batch_topk(np.ones((2, 3), np.float32), rtk.BatchConfig(k=1))


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2409_00822_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h")):
                with open(os.path.join(dirpath, fn)) as f:
                    src = f.read()
                assert not re.search(r"^\s*(import|from)\s+oracle\b", src, re.M), fn
                assert "rtk_oracle" not in src and "librtk_oracle" not in src, fn


def test_file_job_rejects_bad_files_before_touching_the_gpu(lib, tmp_path):
    """rtk_topk_file_f32 validates the RTKM header (io.py:32-43 order) before
    any CUDA call, so these paths run on a CPU box."""
    import struct

    dims = (ctypes.c_int64 * 3)()
    out = str(tmp_path / "o.rtkr").encode()
    rc = lib.rtk_topk_file_f32(str(tmp_path / "missing.rtkm").encode(), out, 1, 0, 0.0, 64, 4, 0, dims)
    assert rc == _native.RTK_EIO
    bad = tmp_path / "bad.rtkm"
    bad.write_bytes(b"NOPE" + b"\x00" * 40)
    assert lib.rtk_topk_file_f32(str(bad).encode(), out, 1, 0, 0.0, 64, 4, 0, dims) == _native.RTK_EFORMAT
    assert b"expected magic b'RTKM'" in lib.rtk_last_error()
    v2 = tmp_path / "v2.rtkm"
    v2.write_bytes(struct.pack("<4sIQQ", b"RTKM", 2, 1, 1) + b"\x00" * 4)
    assert lib.rtk_topk_file_f32(str(v2).encode(), out, 1, 0, 0.0, 64, 4, 0, dims) == _native.RTK_EFORMAT
    tr = tmp_path / "tr.rtkm"
    tr.write_bytes(struct.pack("<4sIQQ", b"RTKM", 1, 4, 4) + b"\x00" * 20)
    assert lib.rtk_topk_file_f32(str(tr).encode(), out, 1, 0, 0.0, 64, 4, 0, dims) == _native.RTK_ETRUNC
    assert (dims[0], dims[1]) == (4, 4)
    short = tmp_path / "short.rtkm"
    short.write_bytes(b"RTKM\x01")
    assert lib.rtk_topk_file_f32(str(short).encode(), out, 1, 0, 0.0, 64, 4, 0, dims) == _native.RTK_ETRUNC
    assert lib.rtk_topk_file_f32(str(tr).encode(), out, 1, 7, 0.0, 64, 4, 0, dims) == _native.RTK_EINVAL
