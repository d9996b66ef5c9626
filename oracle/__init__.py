"""CPU oracle for the row-wise top-k path -- TEST INFRASTRUCTURE ONLY.

A plain-C restatement (``rtk_oracle.c``) of the reference kernels in
``/root/reference/pkg/src/rowtopk/_kernels.py`` plus a ctypes wrapper.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` arm may import this package, and only as the checker or
as the timed CPU baseline; the product package ``paper_2409_00822_b200`` never
imports it.

Parity of the oracle with the reference is pinned against fixtures generated
by importing the reference itself (``tests/golden/make_golden.py``).
"""

from .oracle import (  # noqa: F401
    EXIT_COUNT_EQUALS_K,
    EXIT_DEGENERATE_ROW,
    EXIT_HARD_CAP_REACHED,
    EXIT_INTERVAL_BELOW_EPSILON,
    EXIT_MAX_ITER_REACHED,
    build,
    count_ge,
    early_topk,
    exact_topk,
    exact_trace,
    first_nan_row,
    lib,
    max_threads,
    mid_f32,
    mid_f64,
    mid_mismatches,
    ref_batch,
    row_min_max,
)
