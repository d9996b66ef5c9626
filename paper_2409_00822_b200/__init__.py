"""rowtopk-b200: B200-native row-wise top-k by binary threshold search (RTopK,
arXiv 2409.00822), a drop-in for the reference package's batch entry point
``rowtopk.batch_topk`` (/root/reference/pkg/src/rowtopk/batch.py:105-142).

The compute path is hand-written sm_100a CUDA (csrc/) behind a C ABI
(include/rtk.h, librtk.so) loaded with ctypes; there is no CPU fallback.
"""

__version__ = "1.0.0"

from .batch import (  # noqa: F401
    REGISTER_COLS_LIMIT,
    SOFT_COLS_LIMIT,
    BatchConfig,
    BatchResult,
    as_matrix,
    batch_topk,
    chunk_ranges,
    exact_trace,
    resolve_workers,
    topk_device,
)
from .errors import (  # noqa: F401
    BadMagicError,
    DeviceError,
    DimensionMismatchError,
    EmptyRowError,
    KMismatchError,
    KOutOfRangeError,
    NaNInputError,
    RowTopKError,
    TruncatedFileError,
    VerificationError,
)
from .experiments import (  # noqa: F401
    DataGenSpec,
    EarlyStopStats,
    early_stop_experiment,
    early_stop_grid,
    early_stop_grid_matrix,
    exit_iteration_grid,
    exit_iteration_grid_matrix,
    generate_matrix,
    trial_block,
    trial_row,
)
from .io import load_matrix, load_result, save_matrix, save_result, topk_file  # noqa: F401
from .maxk import (  # noqa: F401
    csr_transpose, gather_rows, maxk, maxk_aggregate, maxk_dense, maxk_dense_fused, maxk_sparse_u8, maxk_spmm,
    scatter_rows, to_sparse_csr)
from .select import (  # noqa: F401
    DEFAULT_HARD_CAP,
    DEFAULT_MAX_ITER,
    ExitReason,
    SearchConfig,
    SearchMode,
    SearchTrace,
    TopKResult,
    as_row,
    count_ge,
    early_stop_topk,
    exact_topk,
    min_max,
    oracle_topk,
)

__all__ = [
    "__version__", "BatchConfig", "BatchResult", "DEFAULT_HARD_CAP", "DEFAULT_MAX_ITER", "DeviceError",
    "DimensionMismatchError", "EmptyRowError", "ExitReason", "KOutOfRangeError", "NaNInputError",
    "REGISTER_COLS_LIMIT", "RowTopKError", "SOFT_COLS_LIMIT", "SearchConfig", "SearchMode", "SearchTrace",
    "TopKResult", "as_matrix", "as_row", "batch_topk", "chunk_ranges", "count_ge", "early_stop_topk",
    "exact_topk", "exact_trace", "min_max", "oracle_topk", "resolve_workers", "load_matrix", "load_result",
    "save_matrix", "save_result", "topk_file", "topk_device", "maxk", "maxk_dense", "maxk_dense_fused", "maxk_sparse_u8", "maxk_spmm", "maxk_aggregate", "csr_transpose", "scatter_rows", "gather_rows", "to_sparse_csr",
    "DataGenSpec", "EarlyStopStats", "early_stop_experiment", "early_stop_grid", "early_stop_grid_matrix",
    "exit_iteration_grid", "exit_iteration_grid_matrix", "generate_matrix", "trial_block", "trial_row",
]
