"""RTKM / RTKR files (io.py mirror) and the native streaming file job
(rtk_topk_file_f32).  Format checks follow the reference's test_io.py
(/root/reference/pkg/tests/test_io.py); the GPU job must write the same bytes
as save_result(batch_topk(load_matrix(path), cfg))."""

import struct

import numpy as np
import pytest

import paper_2409_00822_b200 as rtk
from paper_2409_00822_b200 import io as rio


def _write_rtkm(path, m):
    path.write_bytes(struct.pack("<4sIQQ", b"RTKM", 1, m.shape[0], m.shape[1]) + m.astype("<f4").tobytes())


def test_bad_magic(tmp_path):
    p = tmp_path / "bad.rtkm"
    p.write_bytes(b"NOPE" + b"\x00" * 40)
    with pytest.raises(rtk.BadMagicError):
        rtk.load_matrix(p)


def test_bad_version(tmp_path):
    p = tmp_path / "v2.rtkm"
    p.write_bytes(struct.pack("<4sIQQ", b"RTKM", 2, 1, 1) + b"\x00" * 4)
    with pytest.raises(rtk.BadMagicError, match="version 2"):
        rtk.load_matrix(p)


def test_truncated_header_and_payload(tmp_path):
    p = tmp_path / "short.rtkm"
    p.write_bytes(b"RTKM\x01")
    with pytest.raises(rtk.TruncatedFileError):
        rtk.load_matrix(p)
    q = tmp_path / "trunc.rtkm"
    q.write_bytes(struct.pack("<4sIQQ", b"RTKM", 1, 4, 4) + b"\x00" * (64 - 7))
    with pytest.raises(rtk.TruncatedFileError):
        rtk.load_matrix(q)
    e = tmp_path / "empty.rtkm"
    e.write_bytes(struct.pack("<4sIQQ", b"RTKM", 1, 0, 4))
    with pytest.raises(rtk.TruncatedFileError, match="empty payload"):
        rtk.load_matrix(e)


def test_result_roundtrip_and_layout(tmp_path):
    rng = np.random.default_rng(3)
    res = rtk.BatchResult(values=rng.standard_normal((50, 5)).astype(np.float32),
                          indices=rng.integers(0, 20, (50, 5)).astype(np.int32))
    p = tmp_path / "r.rtkr"
    rtk.save_result(res, p)
    raw = p.read_bytes()
    assert raw[:4] == b"RTKR" and len(raw) == 24 + 50 * 5 * 8
    assert struct.unpack("<IQQ", raw[4:24]) == (1, 50, 5)
    back = rtk.load_result(p)
    assert np.array_equal(back.values, res.values) and np.array_equal(back.indices, res.indices)
    assert back.indices.dtype == np.int32


def test_result_magic_mismatch(tmp_path):
    p = tmp_path / "m.rtkm"
    _write_rtkm(p, np.ones((3, 4), np.float32))
    with pytest.raises(rtk.BadMagicError):
        rtk.load_result(p)


def test_unwritable_result_path_raises_oserror():
    res = rtk.BatchResult(values=np.ones((1, 1), np.float32), indices=np.zeros((1, 1), np.int32))
    with pytest.raises(OSError):
        rtk.save_result(res, "/nonexistent-dir/x.rtkr")


# ----------------------------------------------------------------- GPU job

torch = pytest.importorskip("torch")


@pytest.fixture
def gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2409_00822_b200 import _build

    _build.build()
    torch.cuda.set_device(0)


@pytest.mark.gpu
@pytest.mark.parametrize("n,m,k,search,chunk", [
    (1000, 256, 32, "exact", 0), (1000, 256, 32, "early", 0), (4097, 128, 16, "exact", 300),
    (777, 1024, 64, "early", 100), (333, 97, 97, "exact", 50), (5, 3, 1, "exact", 1), (2049, 512, 200, "exact", 1000),
])
def test_topk_file_matches_oracle_bytes(gpu, oracle_lib, tmp_path, n, m, k, search, chunk):
    rng = np.random.default_rng(n + m)
    x = rng.standard_normal((n, m)).astype(np.float32)
    x[:: max(1, n // 7)] = np.round(x[:: max(1, n // 7)])  # some tie-heavy rows
    src, want, got = tmp_path / "x.rtkm", tmp_path / "want.rtkr", tmp_path / "got.rtkr"
    _write_rtkm(src, x)
    cfg = rtk.BatchConfig(k=k, search=rtk.SearchConfig.exact() if search == "exact" else rtk.SearchConfig.early_stop(3))
    # the expected file is the oracle's result (the reference algorithm on
    # the CPU) written by the reference's save_result layout
    mode = "exact" if search == "exact" else "early"
    v, i, _, _ = oracle_lib.ref_batch(x, k, mode, max_iter=3)
    rtk.save_result(rtk.BatchResult(values=v, indices=i), want)
    assert rtk.topk_file(src, got, cfg, chunk_rows=chunk) == (n, m)
    assert got.read_bytes() == want.read_bytes()


@pytest.mark.gpu
def test_topk_file_reference_digest(gpu, tmp_path):
    """generate_matrix(4096, 256, seed 0) as an RTKM file -> RTKR: values and
    indices equal the reference's digest 5205a48ab4ad5986 (exact) /
    c55e12ced7a981cb (early stop 4)."""
    from golden_util import generate_matrix, h16

    src, got = tmp_path / "x.rtkm", tmp_path / "r.rtkr"
    rtk.save_matrix(generate_matrix(4096, 256, 0), src)
    for search, want in ((rtk.SearchConfig.exact(), "5205a48ab4ad5986"),
                         (rtk.SearchConfig.early_stop(4), "c55e12ced7a981cb")):
        for chunk in (0, 1000):
            assert rtk.topk_file(src, got, rtk.BatchConfig(k=32, search=search), chunk_rows=chunk) == (4096, 256)
            res = rtk.load_result(got)
            assert h16(res.values, res.indices) == want


@pytest.mark.gpu
def test_topk_file_failure_keeps_existing_output(gpu, tmp_path):
    """A failing job leaves an existing result file untouched and no partial
    or temporary file (the reference raises before save_result)."""
    x = np.random.default_rng(2).standard_normal((500, 64)).astype(np.float32)
    x[333, 5] = np.nan
    src, out = tmp_path / "nan.rtkm", tmp_path / "keep.rtkr"
    _write_rtkm(src, x)
    out.write_bytes(b"precious")
    with pytest.raises(rtk.NaNInputError, match="first offending row: 333\\)"):
        rtk.topk_file(src, out, rtk.BatchConfig(k=8), chunk_rows=64)
    assert out.read_bytes() == b"precious"
    assert sorted(p.name for p in tmp_path.iterdir()) == ["keep.rtkr", "nan.rtkm"]


@pytest.mark.gpu
def test_topk_file_error_precedence(gpu, tmp_path):
    out = tmp_path / "o.rtkr"
    cfg = rtk.BatchConfig(k=2)
    with pytest.raises(OSError):
        rtk.topk_file(tmp_path / "missing.rtkm", out, cfg)
    bad = tmp_path / "bad.rtkm"
    bad.write_bytes(b"NOPE" + b"\x00" * 40)
    with pytest.raises(rtk.BadMagicError):
        rtk.topk_file(bad, out, cfg)
    tr = tmp_path / "tr.rtkm"
    tr.write_bytes(struct.pack("<4sIQQ", b"RTKM", 1, 4, 4) + b"\x00" * 20)
    with pytest.raises(rtk.TruncatedFileError):
        rtk.topk_file(tr, out, cfg)
    x = np.random.default_rng(0).standard_normal((100, 16)).astype(np.float32)
    x[61, 3] = np.nan
    x[90, 0] = np.nan
    nanp = tmp_path / "nan.rtkm"
    _write_rtkm(nanp, x)
    with pytest.raises(rtk.NaNInputError, match="first offending row: 61\\)"):
        rtk.topk_file(nanp, out, cfg, chunk_rows=7)
    assert not out.exists()  # no partial result
    with pytest.raises(rtk.NaNInputError):  # NaN before a bad k (batch.py:107-111)
        rtk.topk_file(nanp, out, rtk.BatchConfig(k=17), chunk_rows=7)
    ok = tmp_path / "ok.rtkm"
    _write_rtkm(ok, np.ones((3, 4), np.float32))
    with pytest.raises(rtk.KOutOfRangeError):
        rtk.topk_file(ok, out, rtk.BatchConfig(k=5))
    with pytest.raises(OSError):
        rtk.topk_file(ok, "/nonexistent-dir/o.rtkr", cfg)


@pytest.mark.gpu
def test_matrix_roundtrip_bytes(gpu, tmp_path):
    m = np.random.default_rng(1).standard_normal((17, 9)).astype(np.float32)
    p1, p2 = tmp_path / "a.rtkm", tmp_path / "b.rtkm"
    rtk.save_matrix(m, p1)
    assert p1.stat().st_size == 24 + 17 * 9 * 4
    back = rtk.load_matrix(p1)
    assert np.array_equal(back, m)
    rtk.save_matrix(back, p2)
    assert p1.read_bytes() == p2.read_bytes()
    bad = m.copy()
    bad[4, 2] = np.nan
    q = tmp_path / "nan.rtkm"
    _write_rtkm(q, bad)
    with pytest.raises(rtk.NaNInputError):
        rtk.load_matrix(q)


def test_cli_parser(tmp_path):
    """CLI arguments mirror the reference's `run` / `gen` (cli.py:53-72);
    failures map to the reference's exit codes."""
    from paper_2409_00822_b200 import cli

    a = cli.build_parser().parse_args(["run", "--matrix", "m", "--k", "3", "--out", "o", "--mode", "early-stop"])
    assert (a.k, a.mode, a.max_iter, a.hard_cap, a.workers, a.epsilon_rel) == (3, "early-stop", 4, 64, "auto", 0.0)
    assert cli.build_parser().parse_args(["gen", "--rows", "5", "--cols", "7", "--out", "o"]).seed == 0
    bad = tmp_path / "bad.rtkm"
    bad.write_bytes(b"NOPE" + bytes(20))
    assert cli.main(["run", "--matrix", str(bad), "--k", "1", "--out", str(tmp_path / "o")]) == 3
    # argparse errors are validation errors (1), not argparse's 2 (reference cli.py:35-39)
    assert cli.main(["run", "--matrix", "m", "--k", "x", "--out", "o"]) == 1
    assert cli.main(["run", "--bogus"]) == 1
    assert cli.main([]) == 1
    # file errors come before search validation (reference cli.py:137-141)
    assert cli.main(["run", "--matrix", str(tmp_path / "missing"), "--k", "1", "--max-iter", "0",
                     "--mode", "early-stop", "--out", "o"]) == 3
    tr = tmp_path / "tr.rtkm"
    tr.write_bytes(struct.pack("<4sIQQ", b"RTKM", 1, 4, 4) + bytes(20))
    assert cli.main(["run", "--matrix", str(tr), "--k", "1", "--hard-cap", "0", "--out", "o"]) == 3


@pytest.mark.gpu
def test_cli_run_matches_batch_topk(tmp_path):
    """`run` output bytes == save_result(batch_topk(load_matrix(...))); error
    exit codes as the reference's (3 i/o, 1 validation)."""
    from paper_2409_00822_b200 import cli

    p, out, ref = tmp_path / "x.rtkm", tmp_path / "r.rtkr", tmp_path / "ref.rtkr"
    assert cli.main(["gen", "--rows", "5", "--cols", "7", "--seed", "3", "--out", str(p)]) == 0
    np.testing.assert_array_equal(rtk.load_matrix(p), rtk.generate_matrix(rtk.DataGenSpec(5, 7, seed=3)))
    assert cli.main(["gen", "--rows", "3001", "--cols", "256", "--out", str(p)]) == 0
    for mode in (["--mode", "exact"], ["--mode", "early-stop", "--max-iter", "3"]):
        assert cli.main(["run", "--matrix", str(p), "--k", "32", "--out", str(out), *mode]) == 0
        search = rtk.SearchConfig.exact() if mode[1] == "exact" else rtk.SearchConfig.early_stop(3)
        rtk.save_result(rtk.batch_topk(rtk.load_matrix(p), rtk.BatchConfig(k=32, search=search)), ref)
        assert out.read_bytes() == ref.read_bytes()
    assert cli.main(["run", "--matrix", str(tmp_path / "missing"), "--k", "1", "--out", str(out)]) == 3
    assert cli.main(["run", "--matrix", str(p), "--k", "999", "--out", str(out)]) == 1
    # workers is validated after NaN and k, as batch_topk does (batch.py:106-112)
    assert cli.main(["run", "--matrix", str(p), "--k", "32", "--workers", "0", "--out", str(out)]) == 1
    x = rtk.load_matrix(p).copy()
    x[7, 3] = np.nan
    q = tmp_path / "nan.rtkm"
    _write_rtkm(q, x)
    with pytest.raises(rtk.NaNInputError):
        cli._cmd_run(cli.build_parser().parse_args(["run", "--matrix", str(q), "--k", "999", "--workers", "0",
                                                    "--out", str(out)]))
    with pytest.raises(rtk.KOutOfRangeError):
        cli._cmd_run(cli.build_parser().parse_args(["run", "--matrix", str(p), "--k", "999", "--workers", "0",
                                                    "--out", str(out)]))
