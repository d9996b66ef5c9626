"""CPU: the C oracle (oracle/rtk_oracle.c) is pinned to the reference.

Every golden fixture and every digest in tests/golden/ was produced by the
reference package itself (tests/golden/make_golden.py); the oracle must
reproduce all of them bit for bit before any GPU parity claim is trusted.
"""

import numpy as np
import pytest

from golden_util import cases, digests, generate_matrix, h16, nan_cases


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def test_oracle_matches_every_golden_fixture(oracle_lib):
    n = 0
    for c in cases():
        v, i, t, r = oracle_lib.ref_batch(c["x"], c["k"], c["mode"], max_iter=c["max_iter"] or 4,
                                          eps_rel=c["eps_rel"] or 0.0, hard_cap=c["hard_cap"])
        ctx = (c["xname"], c["k"], c["mode"], c["max_iter"], c["eps_rel"], c["hard_cap"])
        assert np.array_equal(i, c["indices"]), ctx
        assert np.array_equal(_bits(v), _bits(c["values"])), ctx
        assert np.array_equal(t, c["iters"]), ctx
        assert np.array_equal(r, c["reasons"]), ctx
        n += 1
    assert n > 3000


def test_oracle_nan_first_row(oracle_lib):
    for c in nan_cases():
        assert oracle_lib.first_nan_row(c["x"]) == c["first_row"]


@pytest.mark.parametrize("limit", [4096, 65536, 1 << 20])
def test_oracle_matches_reference_digests(oracle_lib, limit):
    """Reference digests at the BASELINE configs (incl. N=2^20 x 256, k=32)."""
    lo = {4096: 0, 65536: 4097, 1 << 20: 65537}[limit]
    checked = 0
    mats = {}
    for c in digests()["cases"]:
        if not (lo <= c["N"] <= limit):
            continue
        key = (c["N"], c["M"], c["seed"])
        if key not in mats:
            mats.clear()
            mats[key] = generate_matrix(c["N"], c["M"], c["seed"])
        x = mats[key]
        assert h16(x) == c["input"], "numpy generator drifted"
        v, i, t, r = oracle_lib.ref_batch(x, c["k"], c["mode"], max_iter=c["max_iter"] or 4,
                                          eps_rel=c["eps_rel"] or 0.0)
        assert h16(v, i) == c["out"], c
        assert h16(t, r) == c["tr"], c
        checked += 1
    assert checked > 0


def test_fp32_midpoint_identity_random_bits(oracle_lib):
    """the float32-only midpoint the kernels use equals the
    reference's F32((F64(a)+F64(b))*0.5) bit for bit."""
    rng = np.random.default_rng(1234)
    n = 2_000_000
    a = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, 1 << 32, n, dtype=np.uint64).astype(np.uint32)
    assert oracle_lib.mid_mismatches(a, b) == 0
    # adjacent floats, subnormals, huge same/opposite sign, and the specials grid
    adj = a.astype(np.uint64) + rng.integers(0, 3, n).astype(np.uint64)
    assert oracle_lib.mid_mismatches(a, (adj & np.uint64(0xFFFFFFFF)).astype(np.uint32)) == 0
    sub = rng.integers(0, 1 << 24, n, dtype=np.uint64).astype(np.uint32)
    sub_b = (rng.integers(0, 1 << 24, n, dtype=np.uint64) | (rng.integers(0, 2, n, dtype=np.uint64) << 31)).astype(np.uint32)
    assert oracle_lib.mid_mismatches(sub, sub_b) == 0
    huge = (0x7E000000 + rng.integers(0, 0x7F800000 - 0x7E000000, n, dtype=np.uint64)).astype(np.uint32)
    huge_b = (0x7E000000 + rng.integers(0, 0x7F800000 - 0x7E000000, n, dtype=np.uint64)).astype(np.uint32)
    assert oracle_lib.mid_mismatches(huge, huge_b) == 0
    assert oracle_lib.mid_mismatches(huge, huge_b | np.uint32(0x80000000)) == 0
    assert oracle_lib.mid_mismatches(huge | np.uint32(0x80000000), huge_b | np.uint32(0x80000000)) == 0
    specials = np.array([0.0, -0.0, np.inf, -np.inf, 1e-45, -1e-45, 1.1754942e-38, 3.4028235e38,
                         -3.4028235e38, 1.0, -1.0, 2e-45], np.float32).view(np.uint32)
    ga, gb = np.meshgrid(specials, specials)
    assert oracle_lib.mid_mismatches(ga.ravel(), gb.ravel()) == 0


def test_oracle_single_row_pieces(oracle_lib):
    assert oracle_lib.row_min_max([3.0, 1.0, 2.0]) == (1.0, 3.0)
    assert oracle_lib.count_ge([1.0, 2.0, 3.0], 2.0) == 2
    assert oracle_lib.count_ge([1.0, 2.0, 3.0], 3.5) == 0


def test_oracle_thread_count_independent(oracle_lib):
    x = generate_matrix(4000, 96, 55)
    ref = oracle_lib.ref_batch(x, 13, "exact", threads=1)
    for th in (2, 3, 8):
        got = oracle_lib.ref_batch(x, 13, "exact", threads=th)
        for a, b in zip(ref, got):
            assert np.array_equal(a, b)
