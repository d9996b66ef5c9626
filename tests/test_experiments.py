"""Experiment drivers against the reference's own
outputs (tests/golden/make_experiments_golden.py ran rowtopk.experiments
on the same trial rows)."""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_2409_00822_b200 as rtk

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "experiments.json")))
ARRAYS = np.load(os.path.join(HERE, "golden", "experiments.npz"))


def test_trial_block_matches_reference_rows():
    """trial rows are the reference's substreams (datagen.py:35-46),
    independent of the host thread split."""
    for m, seed, trials, *_ in GOLD["cases"]:
        spec = rtk.DataGenSpec(1, m, seed=seed)
        for workers in (1, 5):
            block = rtk.trial_block(spec, 0, trials, workers=workers)
            assert hashlib.sha256(block.tobytes()).hexdigest()[:16] == GOLD["inputs"][f"m{m}_s{seed}_t{trials}"]
        np.testing.assert_array_equal(rtk.trial_block(spec, 5, 9), block[5:9])


def test_spec_and_k_validation():
    with pytest.raises(ValueError):
        rtk.DataGenSpec(0, 4)
    with pytest.raises(ValueError):
        rtk.DataGenSpec(1, 0)


@pytest.mark.gpu
def test_exit_iteration_grid_matches_reference():
    """Exit iterations per trial are bit-identical to the reference's."""
    for m, seed, trials, ks, _, epss in GOLD["cases"]:
        spec = rtk.DataGenSpec(1, m, seed=seed)
        for eps in epss:
            grid = rtk.exit_iteration_grid(spec, ks, eps, trials)
            for k in ks:
                want = ARRAYS[f"m{m}_s{seed}_t{trials}_eps{eps!r}_k{k}"]
                np.testing.assert_array_equal(grid[k], want, err_msg=f"m={m} k={k} eps={eps}")


@pytest.mark.gpu
def test_early_stop_grid_matches_reference():
    """Hit rate / E1 / E2 per (k, max_iter) cell equal the reference's up to
    float64 summation order (rel 1e-12); skipped counts exactly."""
    cells = {(c["n_cols"], c["seed"], c["k"], c["max_iter"]): c for c in GOLD["early_stop"]}
    for m, seed, trials, ks, mis, _ in GOLD["cases"]:
        spec = rtk.DataGenSpec(1, m, seed=seed)
        grid = rtk.early_stop_grid(spec, ks, mis, trials)
        for (k, mi), s in grid.items():
            want = cells[(m, seed, k, mi)]
            assert s.trials == trials and s.skipped == want["skipped"]
            for key in ("hit_pct", "e1_pct", "e2_pct"):
                assert getattr(s, key) == pytest.approx(want[key], rel=1e-12, abs=1e-12), (m, k, mi, key)
    one = rtk.early_stop_experiment(rtk.DataGenSpec(1, 256), 32, 4, 3000)
    assert one == rtk.early_stop_grid(rtk.DataGenSpec(1, 256), [32], [4], 3000)[(32, 4)]
    with pytest.raises(rtk.KOutOfRangeError):
        rtk.early_stop_grid(rtk.DataGenSpec(1, 16), [17], [4], 10)


@pytest.mark.gpu
def test_device_rows_grid_at_scale():
    """10^6 device-drawn trials: the early-stop quality grows with max_iter
    and exit iterations stay in the reference's observed range."""
    spec = rtk.DataGenSpec(1, 256, seed=1)
    grid = rtk.early_stop_grid(spec, [32], [2, 4, 8], 1 << 20, device_rows=True)
    hits = [grid[(32, mi)].hit_pct for mi in (2, 4, 8)]
    assert hits[0] < hits[1] < hits[2] <= 100.0
    it = rtk.exit_iteration_grid(spec, [32], 0.0, 1 << 20, device_rows=True)[32]
    assert 7.5 < it.mean() < 9.0
