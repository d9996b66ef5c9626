"""GPU parity: the sm_100a kernels (through the C ABI / public API) against the
reference-generated golden fixtures, the reference digests at BASELINE sizes,
and the C oracle on fresh seeded inputs.  Bit-exact for values (as uint32
bit patterns), indices, trace iterations and trace reasons."""

import numpy as np
import pytest

from conftest import ROW_STYLES, random_row
from golden_util import cases, digests, generate_matrix, h16, nan_cases

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2409_00822_b200 as rtk  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2409_00822_b200 import _build

    _build.build()
    torch.cuda.set_device(0)


def _search(mode, max_iter=None, eps_rel=0.0, hard_cap=64):
    if mode == "exact":
        return rtk.SearchConfig.exact(epsilon_rel=eps_rel or 0.0, hard_cap=hard_cap)
    return rtk.SearchConfig.early_stop(max_iter)


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


def _np(x):
    return x.cpu().numpy() if isinstance(x, torch.Tensor) else x


def _check(res, v, i, t, r, ctx):
    assert np.array_equal(_np(res.indices), i), ctx
    assert np.array_equal(_bits(_np(res.values)), _bits(v)), ctx
    assert np.array_equal(_np(res.trace_iterations), t), ctx
    assert np.array_equal(_np(res.trace_reasons), r), ctx


def test_every_golden_fixture_bit_exact():
    """3000+ reference-generated cases: hand vectors, Appendix B edge rows,
    tie-heavy styles, M = 1..4096, adversarial and special-value rows."""
    n = 0
    for c in cases():
        cfg = rtk.BatchConfig(k=c["k"], search=_search(c["mode"], c["max_iter"], c["eps_rel"], c["hard_cap"]),
                              collect_traces=True)
        res = rtk.batch_topk(c["x"], cfg)  # numpy in -> numpy out (reference calling convention)
        _check(res, c["values"], c["indices"], c["iters"], c["reasons"],
               (c["xname"], c["k"], c["mode"], c["max_iter"], c["eps_rel"], c["hard_cap"]))
        n += 1
    assert n > 3000


def test_golden_fixtures_device_resident_and_strided():
    """Same fixtures through the zero-copy CUDA path with a padded row stride
    (ldx > M) and without traces."""
    for j, c in enumerate(cases()):
        if j % 3:
            continue
        x = c["x"]
        pad = 5 if j % 2 else 4
        buf = torch.full((x.shape[0], x.shape[1] + pad), float("nan"), device="cuda")
        buf[:, : x.shape[1]] = torch.from_numpy(x).cuda()
        view = buf[:, : x.shape[1]]
        cfg = rtk.BatchConfig(k=c["k"], search=_search(c["mode"], c["max_iter"], c["eps_rel"], c["hard_cap"]))
        res = rtk.batch_topk(view, cfg)
        assert res.trace_iterations is None
        assert np.array_equal(res.indices.cpu().numpy(), c["indices"]), c["xname"]
        assert np.array_equal(_bits(res.values.cpu().numpy()), _bits(c["values"])), c["xname"]


def test_nan_rejection_names_first_row():
    for c in nan_cases():
        with pytest.raises(rtk.NaNInputError, match=f"first offending row: {c['first_row']}\\)"):
            rtk.batch_topk(c["x"], rtk.BatchConfig(k=1))
        with pytest.raises(rtk.NaNInputError):
            rtk.batch_topk(torch.from_numpy(c["x"]).cuda(), rtk.BatchConfig(k=1, search=rtk.SearchConfig.early_stop(4)))
        # NaN is reported before a bad k (batch.py:107-111)
        with pytest.raises(rtk.NaNInputError):
            rtk.batch_topk(c["x"], rtk.BatchConfig(k=c["x"].shape[1] + 1))


@pytest.mark.parametrize("limit", [65536, 1 << 20])
def test_reference_digests_at_baseline_sizes(limit):
    """BASELINE configs incl. N=2^20 x 256 k=32 (exact, ES2/4/8), the Reddit
    shape and the M x k sweep: output and trace digests equal the reference's."""
    lo = 0 if limit == 65536 else 65537
    mats = {}
    checked = 0
    for c in digests()["cases"]:
        if not (lo <= c["N"] <= limit):
            continue
        key = (c["N"], c["M"], c["seed"])
        if key not in mats:
            mats.clear()
            x = generate_matrix(c["N"], c["M"], c["seed"])
            assert h16(x) == c["input"]
            mats[key] = torch.from_numpy(x).cuda()
        cfg = rtk.BatchConfig(k=c["k"], search=_search(c["mode"], c["max_iter"], c["eps_rel"]), collect_traces=True)
        res = rtk.batch_topk(mats[key], cfg)
        v, i = res.values.cpu().numpy(), res.indices.cpu().numpy()
        t, r = res.trace_iterations.cpu().numpy(), res.trace_reasons.cpu().numpy()
        assert h16(v, i) == c["out"], c
        assert h16(t, r) == c["tr"], c
        # the hot path (no traces: paired-row / long-row kernels)
        cfg = rtk.BatchConfig(k=c["k"], search=_search(c["mode"], c["max_iter"], c["eps_rel"]))
        res = rtk.batch_topk(mats[key], cfg)
        assert h16(res.values.cpu().numpy(), res.indices.cpu().numpy()) == c["out"], ("no traces", c)
        checked += 1
    assert checked > 0


def test_random_shapes_vs_oracle(oracle_lib):
    rng = np.random.default_rng(77)
    for trial in range(120):
        m = int(rng.choice([int(rng.integers(1, 40)), int(rng.integers(1, 1100)), int(rng.integers(1000, 3000))]))
        n = int(rng.integers(1, 300))
        style = ROW_STYLES[trial % 4]
        x = np.stack([random_row(rng, m, style) for _ in range(n)]) if style != "normal" else \
            rng.standard_normal((n, m), dtype=np.float32) * np.float32(rng.choice([1e-30, 1.0, 1e30]))
        k = int(rng.integers(1, m + 1))
        if trial % 2:
            mode, mi, eps, cap = "exact", 4, float(rng.choice([0.0, 0.0, 1e-16, 1e-3])), int(rng.choice([64, 64, 5]))
        else:
            mode, mi, eps, cap = "early", int(rng.integers(1, 20)), 0.0, 64
        want = oracle_lib.ref_batch(x, k, mode, max_iter=mi, eps_rel=eps, hard_cap=cap)
        res = rtk.batch_topk(x, rtk.BatchConfig(k=k, search=_search(mode, mi, eps, cap), collect_traces=True))
        _check(res, *want, (trial, n, m, k, mode, mi, eps, cap, style))
        res = rtk.batch_topk(x, rtk.BatchConfig(k=k, search=_search(mode, mi, eps, cap)))
        assert np.array_equal(res.indices, want[1]), ("no traces", trial, n, m, k, mode)
        assert np.array_equal(_bits(res.values), _bits(want[0])), ("no traces", trial, n, m, k, mode)


def _mixed_rows(rng, n, m):
    """Rows that take every branch of the fast kernels when processed in
    pairs: N(0,1), tie-heavy styles, constant (degenerate), +-inf, values
    beyond 2^126 (general midpoint), subnormals, duplicated maxima, +-0."""
    kinds = ["normal"] * 6 + ["small-int", "quantized", "constant", "inf", "huge", "tiny", "dupmax", "zeros"]
    rows = []
    for r in range(n):
        kind = kinds[int(rng.integers(len(kinds)))]
        if kind in ("normal", "small-int", "quantized", "constant"):
            row = random_row(rng, m, kind)
        elif kind == "inf":
            row = rng.standard_normal(m).astype(np.float32)
            row[rng.integers(m, size=max(1, m // 50))] = np.float32(np.inf) if r % 2 else np.float32(-np.inf)
        elif kind == "huge":
            row = np.clip(rng.standard_normal(m) * 1.5e38, -3.4e38, 3.4e38).astype(np.float32)
        elif kind == "tiny":
            row = (rng.integers(-20, 21, m) * np.float32(1e-45)).astype(np.float32)
        elif kind == "dupmax":
            row = rng.standard_normal(m).astype(np.float32)
            row[rng.integers(m, size=max(2, m // 8))] = row.max()
        else:
            row = np.where(rng.integers(2, size=m) == 1, np.float32(-0.0), np.float32(0.0)).astype(np.float32)
            row[rng.integers(m, size=3)] = rng.standard_normal(3).astype(np.float32)
        rows.append(row)
    return np.stack(rows)


@pytest.mark.parametrize("m", [4, 8, 100, 128, 200, 256, 260, 384, 500, 512, 640, 768, 1000, 1024, 1025, 1028, 1536,
                               1537, 2048, 2049, 3000, 3072, 3073, 4096, 4097, 6144, 6145, 8192])
def test_fast_paths_mixed_rows_vs_oracle(oracle_lib, m):
    """The no-trace hot paths (paired-row kernel for M <= 256, long-row kernel
    above, masked and unmasked tiles) on odd row counts mixing fast-loop rows
    with rows that need the general per-row path, vs the oracle; then the
    trace path on the same input."""
    rng = np.random.default_rng(1000 + m)
    n = 777 if m <= 256 else (333 if m <= 1024 else 61)
    x = _mixed_rows(rng, n, m)
    ks = sorted({1, min(7, m), min(32, m), max(1, m // 3), max(1, m - 1)})
    searches = [("exact", 4, 0.0, 64), ("exact", 4, 0.0, 7), ("exact", 4, 1e-4, 64), ("early", 2, 0.0, 64),
                ("early", 4, 0.0, 64), ("early", 9, 0.0, 64)]
    for k in ks:
        for mode, mi, eps, cap in searches:
            want = oracle_lib.ref_batch(x, k, mode, max_iter=mi, eps_rel=eps, hard_cap=cap)
            ctx = (m, k, mode, mi, eps, cap)
            res = rtk.batch_topk(x, rtk.BatchConfig(k=k, search=_search(mode, mi, eps, cap)))
            assert np.array_equal(res.indices, want[1]), ctx
            assert np.array_equal(_bits(res.values), _bits(want[0])), ctx
            xd = torch.from_numpy(x).cuda()
            res = rtk.batch_topk(xd, rtk.BatchConfig(k=k, search=_search(mode, mi, eps, cap), collect_traces=True))
            _check(res, *want, ctx)


def test_fast_paths_many_grid_steps_vs_oracle(oracle_lib):
    """Enough rows that every warp of the persistent grid takes many pair /
    ring steps (and an odd tail), device-resident, no traces; sampled rows vs
    the oracle."""
    g = torch.Generator(device="cuda").manual_seed(11)
    for n, m, k in ((300_001, 256, 32), (300_001, 128, 16), (200_001, 256, 128), (200_001, 128, 64),
                    (120_001, 1024, 64), (150_001, 512, 64),
                    (100_003, 768, 128), (20_001, 2048, 64), (30_001, 1500, 64), (12_001, 3072, 128),
                    (10_001, 4000, 64), (9_001, 5000, 64), (9_001, 8192, 256)):
        x = torch.randn(n, m, device="cuda", generator=g)
        rows = torch.tensor([0, 1, 2, 3, n // 3, n // 2 + 1, n - 4, n - 3, n - 2, n - 1], device="cuda")
        xs = x[rows].cpu().numpy()
        for search, mode in ((rtk.SearchConfig.exact(), "exact"), (rtk.SearchConfig.early_stop(4), "early")):
            res = rtk.batch_topk(x, rtk.BatchConfig(k=k, search=search))
            v, i, _, _ = oracle_lib.ref_batch(xs, k, mode, max_iter=4)
            assert np.array_equal(res.indices[rows].cpu().numpy(), i), (n, m, k, mode)
            assert np.array_equal(_bits(res.values[rows].cpu().numpy()), _bits(v)), (n, m, k, mode)
        del x
    torch.cuda.empty_cache()


def test_host_pipeline_chunks_match_device_path(monkeypatch):
    """The chunked H2D -> kernel -> D2H host path (small chunks, pinned and
    pageable inputs, traces on and off) equals the device-resident launch;
    NaN rows are reported with their global row index."""
    from paper_2409_00822_b200 import batch as B

    monkeypatch.setattr(B, "PIPELINE_CHUNK_BYTES", 256 * 1024)
    x = np.random.default_rng(5).standard_normal((10_007, 256), dtype=np.float32)
    for search in (rtk.SearchConfig.exact(), rtk.SearchConfig.early_stop(3)):
        for traces in (False, True):
            cfg = rtk.BatchConfig(k=20, search=search, collect_traces=traces)
            want = rtk.batch_topk(torch.from_numpy(x).cuda(), cfg)
            for host in (x, torch.from_numpy(x).pin_memory()):
                got = rtk.batch_topk(host, cfg)
                assert np.array_equal(got.indices, want.indices.cpu().numpy())
                assert np.array_equal(_bits(got.values), _bits(want.values.cpu().numpy()))
                if traces:
                    assert np.array_equal(got.trace_iterations, want.trace_iterations.cpu().numpy())
                    assert np.array_equal(got.trace_reasons, want.trace_reasons.cpu().numpy())
    x[7000, 3] = np.nan
    x[9000, 3] = np.nan
    with pytest.raises(rtk.NaNInputError, match="first offending row: 7000\\)"):
        rtk.batch_topk(x, rtk.BatchConfig(k=5))


def test_single_row_api_matches_batch_rows():
    """test_batch.py:45-61: every 17th row of 300 x 48 equals the single-row op incl. traces."""
    rng = np.random.default_rng(0xC0FFEE)
    m = rng.standard_normal((300, 48)).astype(np.float32)
    for search in (rtk.SearchConfig.exact(), rtk.SearchConfig.early_stop(3)):
        res = rtk.batch_topk(m, rtk.BatchConfig(k=7, search=search, collect_traces=True))
        traces = res.traces()
        for r in range(0, 300, 17):
            if search.mode is rtk.SearchMode.EXACT:
                single, tr = rtk.exact_topk(m[r], 7)
            else:
                single, tr = rtk.early_stop_topk(m[r], 7, search)
            assert np.array_equal(res.values[r], single.values)
            assert np.array_equal(res.indices[r], single.indices)
            assert traces[r] == tr


def test_single_row_helpers():
    assert rtk.min_max([3.0, 1.0, 2.0]) == (1.0, 3.0)
    assert rtk.min_max([5.0]) == (5.0, 5.0)
    assert rtk.count_ge([1.0, 2.0, 3.0], 2.0) == 2
    assert rtk.count_ge([1.0, 2.0, 3.0], 3.5) == 0
    r = rtk.oracle_topk([1.0, 3.0, 2.0], 2)
    assert r.values.tolist() == [3.0, 2.0] and r.indices.tolist() == [1, 2]
    assert rtk.oracle_topk([5.0, 5.0, 1.0], 1).indices.tolist() == [0]
    with pytest.raises(rtk.EmptyRowError):
        rtk.min_max([])
    with pytest.raises(rtk.NaNInputError):
        rtk.min_max([1.0, float("nan")])
    with pytest.raises(rtk.NaNInputError, match="row contains NaN"):
        rtk.min_max([float("nan"), 2.0, float("inf")])
    with pytest.raises(rtk.NaNInputError, match="row contains NaN"):  # NaN before the k range (select.py:97-112)
        rtk.exact_topk([1.0, float("nan")], 5)
    with pytest.raises(rtk.NaNInputError, match="row contains NaN"):
        rtk.early_stop_topk([float("nan")] * 3, 1, rtk.SearchConfig.early_stop(2))
    with pytest.raises(rtk.NaNInputError):
        rtk.count_ge([1.0], float("nan"))
    with pytest.raises(rtk.KOutOfRangeError):
        rtk.exact_topk([1.0, 2.0], 3)
    with pytest.raises(ValueError):
        rtk.exact_topk([1.0, 2.0], 1, rtk.SearchConfig.early_stop(4))


def test_validation_errors():
    rng = np.random.default_rng(1)
    m = rng.standard_normal((4, 8)).astype(np.float32)
    with pytest.raises(rtk.KOutOfRangeError):
        rtk.batch_topk(m, rtk.BatchConfig(k=9))
    with pytest.raises(rtk.KOutOfRangeError):
        rtk.batch_topk(m, rtk.BatchConfig(k=0))
    with pytest.raises(rtk.DimensionMismatchError):
        rtk.batch_topk(m.ravel(), rtk.BatchConfig(k=2))
    with pytest.raises(rtk.EmptyRowError):
        rtk.batch_topk(np.zeros((0, 4), np.float32), rtk.BatchConfig(k=1))
    with pytest.raises(ValueError):
        rtk.batch_topk(m, rtk.BatchConfig(k=2, workers=0))
    m[2, 5] = np.nan
    with pytest.raises(rtk.NaNInputError, match="row: 2"):
        rtk.batch_topk(m, rtk.BatchConfig(k=2))
    # precedence dims -> NaN -> k -> workers (batch.py:106-112), host and device inputs
    for src in (m, torch.from_numpy(m).cuda()):
        with pytest.raises(rtk.NaNInputError, match="row: 2"):
            rtk.batch_topk(src, rtk.BatchConfig(k=2, workers=0))
        with pytest.raises(rtk.NaNInputError, match="row: 2"):
            rtk.batch_topk(src, rtk.BatchConfig(k=99, workers=0))
    m[2, 5] = 0.0
    for src in (m, torch.from_numpy(m).cuda()):
        with pytest.raises(rtk.KOutOfRangeError):
            rtk.batch_topk(src, rtk.BatchConfig(k=99, workers=0))
        with pytest.raises(ValueError, match="workers"):
            rtk.batch_topk(src, rtk.BatchConfig(k=2, workers=0))


def test_deterministic_and_traces_off_by_default():
    x = torch.randn(4000, 96, device="cuda")
    a = rtk.batch_topk(x, rtk.BatchConfig(k=13, collect_traces=True))
    b = rtk.batch_topk(x, rtk.BatchConfig(k=13, collect_traces=True))
    assert torch.equal(a.values, b.values) and torch.equal(a.indices, b.indices)
    assert torch.equal(a.trace_iterations, b.trace_iterations)
    c = rtk.batch_topk(x, rtk.BatchConfig(k=13))
    assert c.trace_iterations is None
    with pytest.raises(ValueError):
        c.traces()


def test_exact_trace_kernel_matches_oracle(oracle_lib):
    x = generate_matrix(20000, 256, 3)
    for eps in (0.0, 1e-4):
        it, rs = rtk.exact_trace(x, 32, rtk.SearchConfig.exact(epsilon_rel=eps))
        wit, wrs = oracle_lib.exact_trace(x, 32, eps_rel=eps)
        assert np.array_equal(it, wit) and np.array_equal(rs, wrs)


def test_large_offsets_sampled_vs_oracle(oracle_lib):
    """> 2^31 elements in one launch (int64 row offsets), device-generated
    input; a row sample is checked against the oracle."""
    n, m, k = 2_200_000, 1024, 64
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(n, m, device="cuda", generator=g)
    for search, mode in ((rtk.SearchConfig.exact(), "exact"), (rtk.SearchConfig.early_stop(4), "early")):
        res = rtk.batch_topk(x, rtk.BatchConfig(k=k, search=search, collect_traces=True))
        rows = torch.tensor([0, 1, 12345, n // 2, n - 3, n - 2, n - 1], device="cuda")
        xs = x[rows].cpu().numpy()
        v, i, t, r = oracle_lib.ref_batch(xs, k, mode, max_iter=4)
        assert np.array_equal(res.indices[rows].cpu().numpy(), i)
        assert np.array_equal(_bits(res.values[rows].cpu().numpy()), _bits(v))
        assert np.array_equal(res.trace_iterations[rows].cpu().numpy(), t)
    del x
    torch.cuda.empty_cache()


@pytest.mark.parametrize("m", [1, 3, 4, 128, 130, 256])
def test_k_equals_m_copy_paths(m):
    """k == M (_kernels.py:173-179): the row itself with indices 0..M-1 and
    trace (0, DEGENERATE_ROW), on the vectorised copy (M % 4 == 0, aligned)
    and the scalar copy (odd M, strided views, unaligned outputs); NaN rows
    still raise with the first offending row."""
    rng = np.random.default_rng(m)
    n = 70_001
    x = rng.standard_normal((n, m), dtype=np.float32)
    x[5, 0] = -0.0
    want_i = np.broadcast_to(np.arange(m, dtype=np.int32), (n, m))
    for xd in (torch.from_numpy(x).cuda(), torch.from_numpy(np.pad(x, ((0, 0), (0, 3)))).cuda()[:, :m]):
        for search in (rtk.SearchConfig.exact(), rtk.SearchConfig.early_stop(4)):
            res = rtk.batch_topk(xd, rtk.BatchConfig(k=m, search=search, collect_traces=True))
            assert np.array_equal(_bits(_np(res.values)), _bits(x))
            assert np.array_equal(_np(res.indices), want_i)
            assert (_np(res.trace_iterations) == 0).all() and (_np(res.trace_reasons) == 5).all()
    # outputs at an odd ldo through the C ABI (scalar path) and via numpy in
    vals = torch.full((n, m + 1), 7.0, device="cuda")
    idx = torch.full((n, m + 1), -1, dtype=torch.int32, device="cuda")
    xd = torch.from_numpy(x).cuda()
    rtk._native.call("rtk_rowtopk_exact_f32", xd.data_ptr(), n, m, m, m, 0.0, 64, vals.data_ptr(), idx.data_ptr(),
                     m + 1, None, None, None, torch.cuda.current_stream().cuda_stream)
    assert np.array_equal(_bits(vals[:, :m].cpu().numpy()), _bits(x))
    assert np.array_equal(idx[:, :m].cpu().numpy(), want_i)
    assert (vals[:, m] == 7.0).all() and (idx[:, m] == -1).all()
    bad = x.copy()
    bad[n - 3, m - 1] = np.nan
    bad[n - 2, 0] = np.nan
    with pytest.raises(rtk.NaNInputError, match=str(n - 3)):
        rtk.batch_topk(torch.from_numpy(bad).cuda(), rtk.BatchConfig(k=m))


def test_input_dtypes_convert_like_as_matrix(oracle_lib):
    """as_matrix (batch.py:30-36) converts any input to contiguous float32
    before the search: float64 (rounded), float16, integers, bools, nested
    lists, Fortran-ordered arrays, and torch tensors of those dtypes (host and
    CUDA, incl. bfloat16) give the oracle's result on the float32 image."""
    rng = np.random.default_rng(77)
    n, m, k = 1001, 200, 17
    base = rng.standard_normal((n, m)) * 3.0
    inputs = [
        base,  # float64: rounds to nearest float32 like ndarray.astype
        base.astype(np.float16),
        np.round(base * 10).astype(np.int64),
        np.round(base).astype(np.int16),
        base > 0.5,
        np.asfortranarray(base.astype(np.float32)),
        base[:, ::-1],
    ]
    tinputs = [torch.from_numpy(base), torch.from_numpy(base).to(torch.bfloat16),
               torch.from_numpy(base).to(torch.float16), torch.from_numpy(np.round(base * 10).astype(np.int32))]
    for search in (rtk.SearchConfig.exact(), rtk.SearchConfig.early_stop(3)):
        mode = "exact" if search.mode is rtk.SearchMode.EXACT else "early"
        for x in inputs + tinputs + [t.cuda() for t in tinputs] + [base[:5].tolist()]:
            if isinstance(x, torch.Tensor):
                x32 = x.to(torch.float32).cpu().numpy()
            else:
                x32 = np.ascontiguousarray(x, dtype=np.float32)
            want = oracle_lib.ref_batch(x32, k, mode, max_iter=3)
            res = rtk.batch_topk(x, rtk.BatchConfig(k=k, search=search))
            ctx = (type(x).__name__, getattr(x, "dtype", None), mode)
            assert np.array_equal(_np(res.indices), want[1]), ctx
            assert np.array_equal(_bits(_np(res.values)), _bits(want[0])), ctx


def test_long_rows_large_k_shared_memory_fits(oracle_lib):
    """Long rows with k close to M need 8k bytes of staging per warp: the
    launch shrinks the CTA to fit shared memory.  Launches alternate between
    large and small staging on the same kernels (the opt-in size must never
    shrink under a cached launch)."""
    rng = np.random.default_rng(31)
    for m in (1500, 2048, 3000, 4096, 6000, 8192):
        x = rng.standard_normal((37, m), dtype=np.float32)
        for k in (m - 1, 3, m // 2, m):
            for mode in ("exact", "early"):
                want = oracle_lib.ref_batch(x, k, mode, max_iter=4)
                for traces in (True, False):
                    res = rtk.batch_topk(torch.from_numpy(x).cuda(),
                                         rtk.BatchConfig(k=k, search=_search(mode, 4), collect_traces=traces))
                    ctx = (m, k, mode, traces)
                    assert np.array_equal(_np(res.indices), want[1]), ctx
                    assert np.array_equal(_bits(_np(res.values)), _bits(want[0])), ctx


def test_launch_shape_describes_the_dispatch():
    """rtk_launch_shape reports the kernel family the dispatcher picks."""
    import ctypes

    lib = rtk._native.load()

    def shape(m, k, mode):
        w, c, r = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        assert lib.rtk_launch_shape(m, k, mode, ctypes.byref(w), ctypes.byref(c), ctypes.byref(r)) == 0
        return w.value, c.value, r.value

    assert shape(256, 32, 0)[2] == 2 and shape(128, 16, 1)[2] == 2      # paired rows
    assert shape(256, 32, 2)[2] == 1                                      # traces: one row per warp
    for m in (384, 500, 512, 768, 1000, 1024, 2048, 4096):
        w, c, r = shape(m, 64, 0)
        # up to 1024 columns: paired long rows (TMA slots for M = 512 / 1024, the
        # cp.async ring otherwise; exact, and early stop for k < 128 or M > 512)
        assert r == (2 if m <= 1024 else 1) and w >= 1 and c >= 1, (m, w, c, r)
    assert shape(512, 64, 1)[2] == 2 and shape(512, 128, 1)[2] == 1 and shape(512, 64, 2)[2] == 1
    assert shape(1024, 32, 1)[2] == 2 and shape(768, 128, 1)[2] == 2  # early stop, k >= 128: paired above E = 16
    assert shape(8192, 64, 0)[::2] == (2, 0) and shape(8192, 64, 1)[::2] == (4, 0)  # CTA per row
    assert shape(3000, 2999, 1)[0] < 8                                    # large k: fewer warps per CTA
    assert shape(128, 128, 0) == (8, 0, 0)                                # k == M copy


@pytest.mark.parametrize("dtype", ["bfloat16", "float16"])
def test_16bit_rows_native_path(oracle_lib, dtype):
    """bfloat16 / float16 CUDA matrices: M <= 256 rows are read natively by
    rtk_rowtopk_x16 (paired-row kernel, widened in registers), and so are
    256 < M <= 4096 with M % 8 == 0 (long-row kernel, 16-bit ring); results
    equal the oracle's on the float32 image -- the reference's as_matrix
    conversion; other shapes, traces and eps_rel > 0 widen on the device
    first.  Covers masked/unmasked/16-byte/8-byte-aligned tiles, odd N,
    strided views, NaN / inf / huge / tie-heavy rows."""
    tdt = getattr(torch, dtype)
    rng = np.random.default_rng(161)
    for m in (4, 100, 128, 132, 200, 256, 300, 264, 512, 520, 768, 1024, 1032, 2048, 3000, 4096, 5000):
        n = 1001 if m <= 1024 else 203
        x = _mixed_rows(rng, n, m)
        xd = torch.from_numpy(x).cuda().to(tdt)
        x32 = xd.float().cpu().numpy()
        for k in sorted({1, min(16, m - 1) or 1, max(1, m // 3), m - 1, m}):
            for mode, mi, eps in (("exact", 4, 0.0), ("early", 3, 0.0), ("exact", 4, 1e-4)):
                want = oracle_lib.ref_batch(x32, k, mode, max_iter=mi, eps_rel=eps)
                for t in (xd, torch.nn.functional.pad(xd, (0, 8))[:, :m]):  # contiguous, strided (ldx = m + 8)
                    if m > 1024 and t is not xd:
                        continue
                    for traces in (False, True):
                        res = rtk.batch_topk(t, rtk.BatchConfig(k=k, search=_search(mode, mi, eps),
                                                                collect_traces=traces))
                        ctx = (dtype, m, k, mode, eps, traces, t.stride(0))
                        assert res.values.dtype == torch.float32, ctx
                        assert np.array_equal(_np(res.indices), want[1]), ctx
                        assert np.array_equal(_bits(_np(res.values)), _bits(want[0])), ctx
    bad = torch.randn(5000, 256, device="cuda").to(tdt)
    bad[4321, 7] = float("nan")
    with pytest.raises(rtk.NaNInputError, match="4321"):
        rtk.batch_topk(bad, rtk.BatchConfig(k=8))
    # the native entry point itself, and its refusal outside the native shape set
    lib = rtk._native.load()
    x = torch.randn(300_001, 256, device="cuda").to(tdt)
    vals = torch.empty(300_001, 32, device="cuda")
    idx = torch.empty(300_001, 32, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    code = 1 if dtype == "bfloat16" else 2
    assert lib.rtk_rowtopk_x16(x.data_ptr(), code, 1, 300_001, 256, 256, 32, 64, 4, vals.data_ptr(), idx.data_ptr(),
                               32, None, s) == 0
    ref = rtk.batch_topk(x.float(), rtk.BatchConfig(k=32, search=rtk.SearchConfig.early_stop(4)))
    assert torch.equal(vals, ref.values) and torch.equal(idx, ref.indices)
    assert lib.rtk_rowtopk_x16(x.data_ptr(), code, 0, 10, 516, 516, 32, 64, 4, vals.data_ptr(), idx.data_ptr(),
                               32, None, s) == 7  # RTK_EUNSUPPORTED: m > 256 and m % 8 != 0
    assert lib.rtk_rowtopk_x16(x.data_ptr(), code, 0, 10, 5000, 5000, 32, 64, 4, vals.data_ptr(), idx.data_ptr(),
                               32, None, s) == 7  # RTK_EUNSUPPORTED: m > 4096
    assert lib.rtk_rowtopk_x16(x.data_ptr(), 3, 0, 10, 256, 256, 32, 64, 4, vals.data_ptr(), idx.data_ptr(),
                               32, None, s) == 1  # bad dtype


def test_output_row_strides_and_alignment(oracle_lib):
    """Outputs written through the C ABI with row strides that do and do not
    allow 16-byte stores (the paired kernel's vectorised flush for k > 32,
    k % 4 == 0) give the same rows as a contiguous launch; padding columns
    are untouched."""
    rng = np.random.default_rng(9)
    lib = rtk._native.load()
    s = torch.cuda.current_stream().cuda_stream
    for m, k in ((256, 64), (256, 128), (128, 64), (200, 36), (256, 33)):
        x = rng.standard_normal((5001, m), dtype=np.float32)
        xd = torch.from_numpy(x).cuda()
        for mode in ("exact", "early"):
            want = oracle_lib.ref_batch(x, k, mode, max_iter=4)
            for ldo, off in ((k, 0), (k + 4, 0), (k + 2, 0), (k + 4, 1)):
                vals = torch.full((5001 * ldo + 8,), 7.0, device="cuda")
                idx = torch.full((5001 * ldo + 8,), -1, dtype=torch.int32, device="cuda")
                vp, ip = vals[off:].data_ptr(), idx[off:].data_ptr()
                if mode == "exact":
                    rc = lib.rtk_rowtopk_exact_f32(xd.data_ptr(), 5001, m, m, k, 0.0, 64, vp, ip, ldo, None, None,
                                                   None, s)
                else:
                    rc = lib.rtk_rowtopk_early_f32(xd.data_ptr(), 5001, m, m, k, 4, vp, ip, ldo, None, None, None, s)
                assert rc == 0
                v = vals[off:off + 5001 * ldo].view(5001, ldo).cpu().numpy()
                i = idx[off:off + 5001 * ldo].view(5001, ldo).cpu().numpy()
                ctx = (m, k, mode, ldo, off)
                assert np.array_equal(i[:, :k], want[1]), ctx
                assert np.array_equal(_bits(v[:, :k]), _bits(want[0])), ctx
                assert (v[:, k:] == 7.0).all() and (i[:, k:] == -1).all(), ctx


@pytest.mark.parametrize("m", [384, 500, 512, 640, 1000, 1024])
def test_paired_long_rows_adversarial(oracle_lib, m):
    """The paired long-row kernels (TMA slots at M = 512 / 1024, the cp.async
    ring otherwise, masked rows at 500 / 1000) on rows that leave the fast
    loop: tie-heavy and constant rows, ±inf and huge rows (general path in the
    pair), tiny hard caps (finish_exact after the pair loop), odd N (unpaired
    last row), a strided view; exact and early stop (k < 128 paired, k >= 128
    single-row), bit-exact against the oracle."""
    rng = np.random.default_rng(m)
    n = 777
    base = rng.standard_normal((n, m + 12)).astype(np.float32)
    base[1::7] = rng.integers(-2, 3, (len(range(1, n, 7)), m + 12)).astype(np.float32)  # ties at the k-th value
    base[3] = 0.5                                                                      # constant row
    base[10, 5] = np.inf
    base[11, 7] = -np.inf
    base[12, :3] = 3e38                                                                # |max| >= 2^126
    x_host = np.ascontiguousarray(base[:, 4:4 + m])
    xd = torch.from_numpy(base).cuda()[:, 4:4 + m]                                     # strided device view
    for k in (1, 33, 127, 128, m - 1):
        for mode, mi, cap in (("exact", 4, 64), ("exact", 4, 5), ("early", 3, 64), ("early", 9, 64)):
            search = (rtk.SearchConfig.exact(hard_cap=cap) if mode == "exact"
                      else rtk.SearchConfig.early_stop(mi))
            v, i, _, _ = oracle_lib.ref_batch(x_host, k, mode, max_iter=mi, hard_cap=cap)
            res = rtk.batch_topk(xd, rtk.BatchConfig(k=k, search=search))
            assert np.array_equal(res.indices.cpu().numpy(), i), (m, k, mode, mi, cap)
            assert np.array_equal(res.values.cpu().numpy().view(np.uint32), v.view(np.uint32)), (m, k, mode, mi, cap)


@pytest.mark.parametrize("m", [512, 768, 1000, 1024])
def test_long_row_candidate_search_boundaries(oracle_lib, m):
    """The candidate-set exact search of the paired long-row kernels at its
    boundaries: k around the 2-slot / 4-slot / 8-slot / off switches (40, 41,
    96, 97, 192, 193; 8 slots from 16 elements per lane up, its own kernel),
    hard caps small enough to end the search in the full phase, at the switch
    to the candidate phase, or inside it (1..6), and normal rows whose
    candidate set is close to the capacity; bit-exact vs the oracle."""
    rng = np.random.default_rng(7 * m)
    x = rng.standard_normal((401, m)).astype(np.float32)
    x[::9] = np.round(x[::9] * 4) / 4  # coarse values: ties near the k-th value
    for k in (1, 16, 40, 41, 64, 96, 97, 128, 192, 193):
        for cap in (1, 2, 3, 4, 5, 6, 64):
            v, i, _, _ = oracle_lib.ref_batch(x, k, "exact", hard_cap=cap)
            res = rtk.batch_topk(torch.from_numpy(x).cuda(), rtk.BatchConfig(k=k, search=rtk.SearchConfig.exact(hard_cap=cap)))
            assert np.array_equal(res.indices.cpu().numpy(), i), (m, k, cap)
            assert np.array_equal(res.values.cpu().numpy().view(np.uint32), v.view(np.uint32)), (m, k, cap)


@pytest.mark.parametrize("dtype", ["float32", "bfloat16", "float16"])
def test_long_row_paths_fuzz(oracle_lib, dtype):
    """Randomised long rows (257 <= M <= 1024) through every regime of the
    paired long-row kernels -- candidate sets of 2 / 4 / 8 slots and the full
    search above them, hard caps that stop in either phase, early stop, odd N
    (an unpaired last row), masked (M % 32 != 0) and unmasked tiles, mixed
    and tie-heavy rows -- for fp32 and native 16-bit input (compared on the
    float32 image); bit-exact vs the oracle."""
    tdt = getattr(torch, dtype)
    rng = np.random.default_rng({"float32": 5, "bfloat16": 6, "float16": 7}[dtype])
    regimes = [(1, 40), (41, 96), (97, 192), (193, 400)]
    for trial in range(120):
        m = int(rng.choice([int(rng.integers(257, 1025)), int(rng.choice([384, 512, 640, 768, 896, 1024]))]))
        if dtype != "float32":
            m -= m % 8  # the native 16-bit long-row path takes M % 8 == 0
        n = int(rng.integers(1, 120)) * 2 + 1
        x = _mixed_rows(rng, n, m) if trial % 3 else rng.standard_normal((n, m)).astype(np.float32)
        xd = torch.from_numpy(x).cuda().to(tdt)
        x32 = xd.float().cpu().numpy()
        lo, hi = regimes[trial % 4]
        k = int(rng.integers(lo, min(hi, m) + 1))
        if trial % 5 == 4:
            mode, mi, cap = "early", int(rng.integers(1, 9)), 64
        else:
            mode, mi, cap = "exact", 4, int(rng.choice([1, 2, 3, 4, 5, 6, 8, 12, 64, 64, 64]))
        want = oracle_lib.ref_batch(x32, k, mode, max_iter=mi, hard_cap=cap)
        res = rtk.batch_topk(xd, rtk.BatchConfig(k=k, search=_search(mode, mi, 0.0, cap)))
        ctx = (dtype, trial, n, m, k, mode, mi, cap)
        assert np.array_equal(_np(res.indices), want[1]), ctx
        assert np.array_equal(_bits(_np(res.values)), _bits(want[0])), ctx
