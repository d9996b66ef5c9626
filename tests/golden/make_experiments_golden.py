"""Golden outputs of the reference's experiment drivers (rowtopk.experiments,
experiments.py:38-156) for tests/test_experiments.py.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python tests/golden/make_experiments_golden.py

Writes experiments.json (early_stop_grid statistics) and experiments.npz
(exit_iteration_grid arrays).  Nothing here runs at test time.
"""

from __future__ import annotations

import hashlib
import json
import os

import numpy as np

import rowtopk
from rowtopk import DataGenSpec

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = [  # (n_cols, seed, trials, ks, max_iters, epsilons)
    (256, 0, 3000, [16, 32, 64], [1, 2, 4, 8], [0.0, 1e-16, 1e-3]),
    (128, 7, 1500, [16, 128], [2, 4], [0.0]),
    (1024, 3, 600, [64, 1000], [4, 6], [0.0]),
]


def main() -> None:
    stats, arrays, inputs = [], {}, {}
    for m, seed, trials, ks, mis, epss in CASES:
        spec = DataGenSpec(1, m, seed=seed)
        block = rowtopk.trial_block(spec, 0, trials)
        inputs[f"m{m}_s{seed}_t{trials}"] = hashlib.sha256(block.tobytes()).hexdigest()[:16]
        for eps in epss:
            grid = rowtopk.exit_iteration_grid(spec, ks, eps, trials, workers=8)
            for k in ks:
                arrays[f"m{m}_s{seed}_t{trials}_eps{eps!r}_k{k}"] = grid[k]
        grid = rowtopk.early_stop_grid(spec, ks, mis, trials, workers=8)
        for (k, mi), s in grid.items():
            stats.append({"n_cols": m, "seed": seed, "trials": trials, "k": k, "max_iter": mi,
                          "e1_pct": s.e1_pct, "e2_pct": s.e2_pct, "hit_pct": s.hit_pct,
                          "skipped": s.skipped})
    with open(os.path.join(HERE, "experiments.json"), "w") as f:
        json.dump({"cases": CASES, "inputs": inputs, "early_stop": stats}, f, indent=1)
    np.savez_compressed(os.path.join(HERE, "experiments.npz"), **arrays)
    print(len(stats), "grid cells,", len(arrays), "exit arrays")


if __name__ == "__main__":
    main()
