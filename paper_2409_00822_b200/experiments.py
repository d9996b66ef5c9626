"""Repeated-trial experiment drivers on the GPU:
the exit-iteration statistics of the exact search (paper Tables 1/4) and the
early-stop quality grid (Table 2), mirroring the reference's
``rowtopk.experiments`` (/root/reference/pkg/src/rowtopk/experiments.py).

Every trial is one row.  The search and selection of every grid cell run on
the device through the same kernels as ``batch_topk`` (exit statistics via
the traces-only launch, ``exact_trace``); the per-row quality measures are
reduced on the device in float64.

Trial rows.  ``trial_block`` reproduces the reference's data definition
(datagen.py:35-46: trial t is ``default_rng((seed, t)).standard_normal(M,
float32)``), so grids driven by a ``DataGenSpec`` see exactly the
reference's rows; that generation is numpy work on the host.  For 10^6+
trials pass ``device_rows=True``: rows are then drawn on the device from
torch's Philox generator seeded with ``spec.seed`` -- the same distribution,
not the same rows.  The ``*_matrix`` forms take the trial rows directly.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from .batch import _require_cuda, exact_trace, topk_device
from .errors import KOutOfRangeError, NaNInputError
from .select import DEFAULT_HARD_CAP, SearchConfig

DENOMINATOR_GUARD = 1e-12  # metrics.py:14


@dataclass(frozen=True)
class DataGenSpec:
    """datagen.py:21-32 (std-normal rows)."""

    n_rows: int
    n_cols: int
    seed: int = 0

    def __post_init__(self) -> None:
        if self.n_rows < 1:
            raise ValueError(f"n_rows must be >= 1, got {self.n_rows}")
        if self.n_cols < 1:
            raise ValueError(f"n_cols must be >= 1, got {self.n_cols}")


@dataclass(frozen=True)
class EarlyStopStats:
    """metrics.py:17-25: aggregates over an early-stop experiment, in percent."""

    e1_pct: float
    e2_pct: float
    hit_pct: float
    trials: int
    skipped: int


def trial_row(spec: DataGenSpec, trial: int) -> np.ndarray:
    """Row of one trial from the substream (seed, trial) (datagen.py:35-38)."""
    return np.random.default_rng((spec.seed, trial)).standard_normal(spec.n_cols, dtype=np.float32)


def trial_block(spec: DataGenSpec, start: int, stop: int, workers: int = 0) -> np.ndarray:
    """Rows of trials [start, stop) stacked into a (stop-start, M) matrix
    (datagen.py:41-46); generated on `workers` host threads (0: all cores)."""
    n = stop - start
    block = np.empty((n, spec.n_cols), np.float32)
    workers = workers or min(32, os.cpu_count() or 1)

    def fill(a: int, b: int) -> None:
        for t in range(a, b):
            block[t - start] = trial_row(spec, t)

    step = max(256, -(-n // workers))
    spans = [(a, min(a + step, stop)) for a in range(start, stop, step)]
    if len(spans) <= 1:
        for a, b in spans:
            fill(a, b)
    else:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            list(pool.map(lambda ab: fill(*ab), spans))
    return block


def generate_matrix(spec: DataGenSpec) -> np.ndarray:
    """Full N x M matrix from one stream keyed by the seed (datagen.py:49-52)."""
    return np.random.default_rng(spec.seed).standard_normal((spec.n_rows, spec.n_cols), dtype=np.float32)


def _trial_rows(spec: DataGenSpec, trials: int, device_rows: bool):
    torch = _require_cuda()
    if trials < 1:
        raise ValueError(f"trials must be >= 1, got {trials}")
    if device_rows:
        g = torch.Generator(device="cuda")
        g.manual_seed(int(spec.seed))
        return torch.randn((trials, spec.n_cols), generator=g, device="cuda", dtype=torch.float32)
    return torch.from_numpy(trial_block(spec, 0, trials)).cuda()


def _check_ks(ks, m: int) -> None:
    for k in ks:
        if not 1 <= k <= m:
            raise KOutOfRangeError(f"k must be in [1, {m}], got {k}")


def exit_iteration_grid_matrix(x, ks: list[int], epsilon_rel: float, hard_cap: int = DEFAULT_HARD_CAP):
    """Exit iterations of the exact search per k over the rows of x (a CUDA
    float32 matrix): {k: int32 CUDA tensor (N,)} (experiments.py:38-66)."""
    _check_ks(ks, int(x.shape[1]))
    search = SearchConfig.exact(epsilon_rel=float(epsilon_rel), hard_cap=int(hard_cap))
    return {k: exact_trace(x, k, search)[0] for k in ks}


def exit_iteration_grid(spec: DataGenSpec, ks: list[int], epsilon_rel: float, trials: int,
                        hard_cap: int = DEFAULT_HARD_CAP, workers: int = 1,
                        device_rows: bool = False) -> dict[int, np.ndarray]:
    """experiments.py:38-66: {k: int32 array of length trials}.  `workers` is
    accepted for signature parity (the search runs on the GPU)."""
    _check_ks(ks, spec.n_cols)
    x = _trial_rows(spec, trials, device_rows)
    return {k: it.cpu().numpy() for k, it in exit_iteration_grid_matrix(x, ks, epsilon_rel, hard_cap).items()}


def _optimal_mask(x, k: int):
    """Membership of the first k columns of a stable descending argsort
    (experiments.py:72,75-78): everything above the k-th largest value plus
    the lowest-index ties at it; and the k-th largest value itself."""
    torch = _require_cuda()
    kth = torch.topk(x, k, dim=1, sorted=True).values[:, k - 1 : k]
    greater = x > kth
    need = k - greater.sum(dim=1, keepdim=True)
    eq = x == kth
    rank = torch.cumsum(eq.to(torch.int32), dim=1)
    return greater | (eq & (rank <= need)), kth[:, 0]


def _quality_sums(x, opt, opt_min, row_max, skip, k: int, max_iter: int):
    """(hit_sum, e1_sum, e2_sum) of the early-stop selection with max_iter
    against the optimal selection (experiments.py:80-100), in float64."""
    torch = _require_cuda()
    nan_word = torch.empty(1, dtype=torch.int32, device=x.device)
    vals, idx = topk_device(x, k, SearchConfig.early_stop(int(max_iter)), nan_word=nan_word)
    r = int(nan_word.item())
    if r != -1:
        raise NaNInputError(f"matrix contains NaN (first offending row: {r & 0xFFFFFFFF})")
    hit = torch.gather(opt, 1, idx.long()).sum(dim=1).to(torch.float64) / k
    e1 = (vals.max(dim=1).values.to(torch.float64) - row_max).abs() / row_max.abs()
    e2 = (vals.min(dim=1).values.to(torch.float64) - opt_min).abs() / opt_min.abs()
    keep = ~skip
    return hit.sum().item(), e1[keep].sum().item(), e2[keep].sum().item()


def early_stop_grid_matrix(x, ks: list[int], max_iters: list[int]) -> dict[tuple[int, int], EarlyStopStats]:
    """Early-stop quality vs the optimal selection over a (k, max_iter) grid
    on the rows of x (CUDA float32), as experiments.py:103-149 reports it:
    hit averaged over all rows, E1/E2 over rows whose reference extremes pass
    the denominator guard (the rest counted as skipped)."""
    torch = _require_cuda()
    trials, m = int(x.shape[0]), int(x.shape[1])
    _check_ks(ks, m)
    if trials < 1:
        raise ValueError(f"trials must be >= 1, got {trials}")
    row_max = x.max(dim=1).values.to(torch.float64)
    stats = {}
    for k in ks:
        opt, kth = _optimal_mask(x, k)
        opt_min = kth.to(torch.float64)
        skip = (row_max.abs() < DENOMINATOR_GUARD) | (opt_min.abs() < DENOMINATOR_GUARD)
        skipped = int(skip.sum().item())
        used = trials - skipped
        for mi in max_iters:
            hit_sum, e1_sum, e2_sum = _quality_sums(x, opt, opt_min, row_max, skip, k, mi)
            stats[(k, mi)] = EarlyStopStats(
                e1_pct=(e1_sum / used * 100.0) if used else float("nan"),
                e2_pct=(e2_sum / used * 100.0) if used else float("nan"),
                hit_pct=hit_sum / trials * 100.0,
                trials=trials,
                skipped=skipped,
            )
    return stats


def early_stop_grid(spec: DataGenSpec, ks: list[int], max_iters: list[int], trials: int, workers: int = 1,
                    device_rows: bool = False) -> dict[tuple[int, int], EarlyStopStats]:
    """experiments.py:103-149 on the GPU (`workers` accepted for signature parity)."""
    _check_ks(ks, spec.n_cols)
    return early_stop_grid_matrix(_trial_rows(spec, trials, device_rows), ks, max_iters)


def early_stop_experiment(gen: DataGenSpec, k: int, max_iter: int, trials: int, workers: int = 1,
                          device_rows: bool = False) -> EarlyStopStats:
    """Single-cell wrapper around early_stop_grid (experiments.py:152-156)."""
    return early_stop_grid(gen, [k], [max_iter], trials, workers, device_rows)[(k, max_iter)]
