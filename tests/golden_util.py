"""Readers for the committed golden fixtures (tests/golden/, made by make_golden.py
from the reference itself).  No reference code is needed at test time."""

from __future__ import annotations

import functools
import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def h16(*arrays) -> str:
    m = hashlib.sha256()
    for a in arrays:
        m.update(np.ascontiguousarray(a).tobytes())
    return m.hexdigest()[:16]


@functools.lru_cache(maxsize=1)
def fixtures():
    z = np.load(os.path.join(GOLDEN, "fixtures.npz"))
    data = {k: z[k] for k in z.files}
    meta = json.loads(bytes(data.pop("meta")).decode())
    return data, meta


def cases():
    """Yield dicts: x, k, mode, max_iter, eps_rel, hard_cap, tag, values, indices, iters, reasons."""
    data, meta = fixtures()
    for c in meta["cases"]:
        x = data["x_" + c["x"]]
        idx = data[f"i_{c['id']}"]
        vals = np.take_along_axis(x, idx.astype(np.int64), axis=1)
        yield dict(c, x=x, xname=c["x"], values=vals, indices=idx,
                   iters=data[f"t_{c['id']}"], reasons=data[f"r_{c['id']}"])


def nan_cases():
    data, meta = fixtures()
    for c in meta["nan"]:
        yield dict(c, x=data["x_" + c["x"]])


@functools.lru_cache(maxsize=1)
def digests():
    with open(os.path.join(GOLDEN, "digests.json")) as f:
        return json.load(f)


def generate_matrix(n: int, m: int, seed: int) -> np.ndarray:
    """The reference generator (datagen.py:49-52)."""
    return np.random.default_rng(seed).standard_normal((n, m), dtype=np.float32)
