"""Generate the golden fixtures for the row-wise top-k path FROM THE REFERENCE.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python tests/golden/make_golden.py

It imports the reference package ``rowtopk`` and records
  * digests.json   -- sha256[:16] digests of inputs/outputs/traces of
                      reference ``batch_topk`` on the BASELINE.json configs
                      (values+indices bytes, and iterations+reasons bytes);
  * fixtures.npz   -- full inputs, output indices and traces for small cases
                      (output values are x[row, idx] bit copies, asserted
                      here, so they are not stored): the reference
                      test suite's hand vectors, SURVEY Appendix B edge rows,
                      the tie-heavy styles of verify._style_matrix /
                      conftest.random_row, hypothesis-style adversarial rows,
                      special-value rows (+-inf, +-0, subnormals, huge), and
                      every M from 1 to beyond the register path's 1024 limit.
Nothing here runs at test time; tests only read the committed files.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

import rowtopk
from rowtopk import BatchConfig, DataGenSpec, SearchConfig, batch_topk, generate_matrix
from rowtopk.errors import NaNInputError

HERE = os.path.dirname(os.path.abspath(__file__))


def h16(*arrays) -> str:
    m = hashlib.sha256()
    for a in arrays:
        m.update(np.ascontiguousarray(a).tobytes())
    return m.hexdigest()[:16]


def run(x, k, mode, param=None, eps_rel=0.0, hard_cap=64, workers="auto"):
    if mode == "exact":
        search = SearchConfig.exact(epsilon_rel=eps_rel, hard_cap=hard_cap)
    else:
        search = SearchConfig.early_stop(param)
    return batch_topk(x, BatchConfig(k=k, search=search, workers=workers, collect_traces=True))


def digests():
    out = {"format": "sha256(values.tobytes()+indices.tobytes())[:16]; tr = sha256(iters+reasons)[:16]",
           "generator": "numpy.random.default_rng(seed).standard_normal((N, M), dtype=float32)",
           "numpy": np.__version__, "reference": rowtopk.__version__, "cases": []}
    cfgs = [
        (4096, 256, 32, 0), (4096, 256, 32, 987), (1 << 20, 256, 32, 0), (232965, 256, 32, 0),
        (65536, 1024, 128, 0), (65536, 128, 16, 0),
    ]
    for M in (128, 256, 512, 768, 1024):
        for k in (16, 32, 64, 128):
            cfgs.append((65536, M, k, 0))
    seen = set()
    for (N, M, k, seed) in cfgs:
        if (N, M, k, seed) in seen:
            continue
        seen.add((N, M, k, seed))
        x = generate_matrix(DataGenSpec(N, M, seed=seed))
        modes = [("exact", None, 0.0), ("early", 4, None)]
        if N in (4096, 1 << 20, 232965) or (N, M, k) in ((65536, 1024, 128), (65536, 128, 16)):
            modes += [("early", 2, None), ("early", 8, None)]
        if N == 4096:
            modes += [("exact", None, 1e-16), ("exact", None, 1e-4)]
        for mode, mi, eps in modes:
            r = run(x, k, mode, mi, eps_rel=eps or 0.0)
            out["cases"].append({
                "N": N, "M": M, "k": k, "seed": seed, "mode": mode, "max_iter": mi,
                "eps_rel": eps, "input": h16(x), "out": h16(r.values, r.indices),
                "tr": h16(r.trace_iterations, r.trace_reasons),
                "reasons_hist": np.bincount(r.trace_reasons, minlength=6).tolist(),
            })
            print(out["cases"][-1], flush=True)
    return out


F32 = np.float32


def special_rows(rng, m, n):
    pool = np.array([np.inf, -np.inf, 0.0, -0.0, 1.0, -1.0, 3.4e38, -3.4e38, 1e-45, -1e-45, 2e-45,
                     1.1754942e-38, 1e-30, 2e-30, -1e-30, 5.0, 5.0, 9.0, 1e6, -1e6], np.float64).astype(F32)
    return pool[rng.integers(0, pool.size, (n, m))]


def adversarial_rows(rng, m, n):
    pool = np.array([-2.5, -1.0, -0.0, 0.0, 0.25, 1.0, 1.0, 3.5, 1e6, -1e6], np.float64).astype(F32)
    cont = rng.uniform(-1e6, 1e6, (n, m)).astype(F32)
    pick = rng.integers(0, pool.size, (n, m))
    use_pool = rng.random((n, m)) < 0.5
    return np.where(use_pool, pool[pick], cont).astype(F32)


def style_matrix(rng, style, n, m):
    if style == "normal":
        return rng.standard_normal((n, m), dtype=F32)
    if style == "small-int":
        return rng.integers(-3, 4, (n, m)).astype(F32)
    if style == "quantized":
        return np.round(rng.standard_normal((n, m)) * 4.0).astype(F32) / F32(4.0)
    if style == "constant":
        return np.repeat(rng.standard_normal((n, 1)).astype(F32), m, axis=1)
    raise ValueError(style)


def fixtures():
    arrays = {}
    meta = []
    mats = {}

    def add_matrix(name, x):
        x = np.ascontiguousarray(x, F32)
        arrays[f"x_{name}"] = x
        mats[name] = x
        return name

    def add_case(xname, k, mode, param=None, eps_rel=0.0, hard_cap=64, tag=""):
        x = mats[xname]
        r = run(x, k, mode, param, eps_rel=eps_rel, hard_cap=hard_cap)
        i = len(meta)
        # values are bit copies of x[row, idx] (_kernels.py:122,142); store indices only
        assert np.array_equal(np.take_along_axis(x, r.indices.astype(np.int64), axis=1).view(np.uint32),
                              r.values.view(np.uint32))
        arrays[f"i_{i}"] = r.indices
        arrays[f"t_{i}"] = r.trace_iterations
        arrays[f"r_{i}"] = r.trace_reasons
        meta.append({"id": i, "x": xname, "k": int(k), "mode": mode, "max_iter": param,
                     "eps_rel": eps_rel, "hard_cap": hard_cap, "tag": tag})

    # reference test-suite hand vectors (test_batch.py:53-57, test_select.py:244-305)
    add_matrix("hand23", [[3, 1, 2], [0, 5, 4]])
    add_case("hand23", 2, "exact", tag="test_batch.py:53")
    for j, (row, k, hc) in enumerate([([3.0, 1.0, 2.0], 3, 64), ([0.5, 2.0, -1.0], 1, 64),
                                      ([7.0, 7.0, 7.0, 7.0], 2, 64), ([5.0, 5.0, 9.0], 2, 64),
                                      ([9.0, 9.0, 9.0, 1.0], 2, 64), ([1.0, 5.0, 5.0, 5.0, 9.0], 3, 64),
                                      ([5.0, 5.0, 9.0], 2, 3), ([7.0, 7.0, 7.0], 2, 64)]):
        name = add_matrix(f"hand_{j}", [row])
        add_case(name, k, "exact", hard_cap=hc, tag="test_select.py")
        add_case(name, k, "early", 4, tag="test_select.py")

    # SURVEY.md Appendix B edge rows (exact eps 0, eps 1e-4 and ES4)
    edge = [([1, np.inf, 3, 2], 2), ([1, np.inf, np.inf, 2], 1), ([-np.inf, 1, 3, 2], 2),
            ([-np.inf, 1, np.inf, 2], 2), ([0.0, -0.0, 0.0, -0.0], 2), ([-0.0, 1, 0.0, -1], 2),
            (list(np.array([1e-45, 0, 2e-45, -1e-45], F32)), 2),
            ([-1e6, 1e6, 0, 1e-30, 2e-30, 3e-30, -1e-30], 3), ([-1e6, 1e6, 0, 1e-30, 2e-30, 3e-30, -1e-30], 5),
            ([-3.4e38, 3.4e38, 1, 2], 2), ([3.4e38, 3.4e38, 3.3e38, 1], 2), ([-3.4e38, -3.4e38, 1, -3.3e38], 3),
            ([np.inf, -np.inf, np.inf, -np.inf], 2), ([-np.inf, -np.inf, -np.inf, 0], 1)]
    for j, (row, k) in enumerate(edge):
        name = add_matrix(f"edge_{j}", np.array([row], np.float64).astype(F32))
        add_case(name, k, "exact", tag="appendixB")
        add_case(name, k, "exact", eps_rel=1e-4, tag="appendixB")
        for mi in (1, 4, 9):
            add_case(name, k, "early", mi, tag="appendixB")

    # every register-path shape class: M in 1..33, around 128-multiples, up to 1024 and beyond
    rng = np.random.default_rng(20240901)
    ms = list(range(1, 34)) + [47, 48, 63, 64, 65, 96, 97, 127, 128, 129, 131, 192, 255, 256, 257, 300,
                               383, 384, 511, 512, 513, 640, 767, 768, 769, 896, 1000, 1023, 1024,
                               1025, 1536, 2048, 3001, 4096]
    for m in ms:
        n = 48 if m <= 64 else (16 if m <= 256 else (6 if m <= 1024 else 3))
        for style in ("normal", "small-int", "quantized", "constant"):
            if style == "constant" and m not in (1, 7, 64, 97, 256, 1000, 1025):
                continue
            name = add_matrix(f"s_{style}_{m}", style_matrix(rng, style, n, m))
            ks = sorted({1, 2, max(1, m // 8), max(1, m // 4), max(1, m // 2), max(1, m - 1), m})
            if m > 64:
                ks = sorted({1, 2, max(1, m // 8), max(1, m // 4), m - 1 if m <= 130 else m // 3} | ({m} if m <= 300 else set()))
            ks = [k for k in ks if 1 <= k <= m]
            for k in ks:
                add_case(name, k, "exact", tag="style")
                if k in (max(1, m // 4), 1, m):
                    add_case(name, k, "early", 4, tag="style")
                if k == max(1, m // 8):
                    add_case(name, k, "early", 1, tag="style")
                    add_case(name, k, "early", 11, tag="style")
                    add_case(name, k, "exact", eps_rel=0.05, tag="style")
                    add_case(name, k, "exact", hard_cap=3, tag="style")
                    add_case(name, k, "exact", eps_rel=1e-16, tag="style")

    # hypothesis-style adversarial rows (test_select_properties.py:14-19)
    for m in list(range(2, 25)) + [100, 256, 260]:
        name = add_matrix(f"adv_{m}", adversarial_rows(rng, m, 40))
        for k in sorted({1, max(1, m // 3), max(1, m - 1)}):
            add_case(name, k, "exact", tag="adversarial")
            add_case(name, k, "early", int(rng.integers(1, 17)), tag="adversarial")
    # special-value rows (+-inf, +-0, subnormals, huge)
    for m in (2, 3, 5, 8, 16, 37, 128, 256, 300):
        name = add_matrix(f"sp_{m}", special_rows(rng, m, 64))
        for k in sorted({1, max(1, m // 2), max(1, m - 1)}):
            add_case(name, k, "exact", tag="special")
            add_case(name, k, "exact", eps_rel=1e-4, tag="special")
            add_case(name, k, "exact", hard_cap=5, tag="special")
            add_case(name, k, "early", 4, tag="special")
            add_case(name, k, "early", 30, tag="special")
    # the reference test_batch.py:68-84 shape (300 x 48, k=7, exact / ES3)
    x = np.random.default_rng(0xC0FFEE).standard_normal((300, 48)).astype(F32)
    add_matrix("batch300x48", x)
    add_case("batch300x48", 7, "exact", tag="test_batch.py:68")
    add_case("batch300x48", 7, "early", 3, tag="test_batch.py:68")

    # NaN rejection (batch.py:37-39): expected first offending row
    nan_cases = []
    for j, (n, m, rows) in enumerate([(4, 8, [2]), (10, 256, [7, 3]), (1, 1, [0]), (64, 97, [63])]):
        x = np.random.default_rng(j).standard_normal((n, m)).astype(F32)
        for r in rows:
            x[r, (r * 7) % m] = np.nan
        name = add_matrix(f"nan_{j}", x)
        try:
            batch_topk(x, BatchConfig(k=1))
            raise SystemExit("reference accepted NaN input?")
        except NaNInputError as e:
            msg = str(e)
        nan_cases.append({"x": name, "message": msg, "first_row": int(msg.split(":")[-1].strip(" )"))})
    return arrays, meta, nan_cases


def main():
    arrays, meta, nan_cases = fixtures()
    arrays["meta"] = np.frombuffer(json.dumps({"cases": meta, "nan": nan_cases}).encode(), np.uint8)
    np.savez_compressed(os.path.join(HERE, "fixtures.npz"), **arrays)
    print("fixture cases:", len(meta), "bytes:", os.path.getsize(os.path.join(HERE, "fixtures.npz")))
    if "--no-digests" not in sys.argv:
        d = digests()
        with open(os.path.join(HERE, "digests.json"), "w") as f:
            json.dump(d, f, indent=1)


if __name__ == "__main__":
    main()
