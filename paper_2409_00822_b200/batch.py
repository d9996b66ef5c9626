"""Row-parallel engine on the B200: the drop-in for rowtopk.batch_topk.

Mirrors /root/reference/pkg/src/rowtopk/batch.py (BatchConfig, BatchResult,
as_matrix, resolve_workers, chunk_ranges, batch_topk) with the same
validation order and messages:

    dimension / empty (batch.py:33-36) -> NaN (batch.py:37-39)
    -> k range (batch.py:110-111) -> workers (batch.py:112)

The reference splits rows into contiguous chunks for a CPU thread pool
(batch.py:87-102).  Here the whole matrix goes to one persistent sm_100a
kernel launch through the C ABI (include/rtk.h); the NaN scan is fused into
that launch and reported through a device word read back after the stream
completes.  `workers` is validated and otherwise ignored.  Host inputs
(numpy / lists / CPU tensors) are copied to the current CUDA device and the
results come back as numpy arrays; CUDA tensors are used in place (any row
stride) and the results stay on their device as torch tensors.
"""

from __future__ import annotations

import os
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import DeviceError, DimensionMismatchError, EmptyRowError, KOutOfRangeError, NaNInputError
from .select import ExitReason, SearchConfig, SearchMode, SearchTrace

# batch.py:27 -- the validated regime of the paper's GPU analysis (not enforced).
SOFT_COLS_LIMIT = 8192
# Rows up to this length run from registers; longer rows from L1/L2 (rtk_kernels.cuh).
REGISTER_COLS_LIMIT = 1024


def _torch():
    import torch

    return torch


def _require_cuda():
    torch = _torch()
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device is visible; rowtopk-b200 has no CPU fallback")
    return torch


def _is_torch(x) -> bool:
    try:
        torch = _torch()
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def _host_matrix(values) -> np.ndarray:
    """The conversion + shape checks of as_matrix (batch.py:30-36), on the host."""
    if _is_torch(values):
        torch = _torch()
        t = values.detach()
        if t.dtype == torch.bfloat16:  # no numpy dtype; the widening to float32 is exact
            t = t.to(torch.float32)
        values = t.cpu().numpy()
    m = np.ascontiguousarray(values, dtype=np.float32)
    if m.ndim != 2:
        raise DimensionMismatchError(f"expected a 2-D matrix, got shape {m.shape}")
    if m.shape[0] == 0 or m.shape[1] == 0:
        raise EmptyRowError(f"matrix must be at least 1 x 1, got {m.shape}")
    return m


class _DeviceMatrix:
    """A validated-shape float32 matrix resident on a CUDA device, plus the
    launch helpers over the C ABI.  Holds the host origin (if any) so results
    can be returned in the caller's array type."""

    def __init__(self, values):
        torch = _require_cuda()
        self._x = None
        self.x16 = None
        self.host = not (_is_torch(values) and values.is_cuda)
        if self.host:
            if _is_torch(values) and values.dim() == 2 and values.dtype == torch.float32:
                t = values if values.is_contiguous() else values.contiguous()
                if t.numel() == 0:
                    raise EmptyRowError(f"matrix must be at least 1 x 1, got {tuple(t.shape)}")
            else:
                with warnings.catch_warnings():  # read-only arrays (memmaps) are only read from
                    warnings.simplefilter("ignore", UserWarning)
                    t = torch.from_numpy(_host_matrix(values))
            self._x = t.to(torch.device("cuda", torch.cuda.current_device()),
                           non_blocking=t.is_pinned())
        else:
            t = values
            if t.dim() != 2:
                raise DimensionMismatchError(f"expected a 2-D matrix, got shape {tuple(t.shape)}")
            if t.shape[0] == 0 or t.shape[1] == 0:
                raise EmptyRowError(f"matrix must be at least 1 x 1, got {tuple(t.shape)}")
            if t.dtype in (torch.bfloat16, torch.float16) and t.stride(1) == 1 and (
                    t.shape[0] == 1 or t.stride(0) >= t.shape[1]):
                # kept as is: the top-k launch reads 16-bit rows natively where
                # it can (rtk_rowtopk_x16); other uses widen on first access
                self.x16 = t
            else:
                if t.dtype != torch.float32:
                    t = t.to(torch.float32)
                if t.stride(1) != 1 or (t.shape[0] > 1 and t.stride(0) < t.shape[1]):
                    t = t.contiguous()
                self._x = t
        src = self._x if self._x is not None else self.x16
        self.n, self.m = int(src.shape[0]), int(src.shape[1])
        self.device = src.device

    @property
    def x(self):
        """The matrix as float32 on the device (16-bit inputs are widened --
        exactly -- on first use, as as_matrix does, batch.py:30-36)."""
        if self._x is None:
            self._x = self.x16.to(_torch().float32).contiguous()
        return self._x

    @property
    def ldx(self) -> int:
        return int(self.x.stride(0)) if self.n > 1 else self.m

    # -- plumbing
    def _stream(self):
        torch = _torch()
        return torch.cuda.current_stream(self.device).cuda_stream

    def _new_nan_word(self):
        torch = _torch()
        return torch.empty(1, dtype=torch.int32, device=self.device)

    @staticmethod
    def _nan_row(word) -> int:
        v = int(word.item())  # device -> host read; syncs the stream
        return -1 if v == -1 else v & 0xFFFFFFFF

    # -- operations
    def first_nan_row(self) -> int:
        """Device NaN scan (batch.py:37-39); -1 when the matrix is NaN-free."""
        word = self._new_nan_word()
        with _torch().cuda.device(self.device):
            _native.call("rtk_nan_scan_f32", self.x.data_ptr(), self.n, self.m, self.ldx,
                         word.data_ptr(), self._stream())
        return self._nan_row(word)

    def row_min_max(self):
        torch = _torch()
        mins = torch.empty(self.n, dtype=torch.float32, device=self.device)
        maxs = torch.empty(self.n, dtype=torch.float32, device=self.device)
        with torch.cuda.device(self.device):
            _native.call("rtk_row_min_max_f32", self.x.data_ptr(), self.n, self.m, self.ldx,
                         mins.data_ptr(), maxs.data_ptr(), self._stream())
        return mins.cpu().numpy(), maxs.cpu().numpy()

    def count_ge(self, thres):
        torch = _torch()
        t = torch.as_tensor(np.ascontiguousarray(thres, np.float32)).to(self.device)
        counts = torch.empty(self.n, dtype=torch.int32, device=self.device)
        with torch.cuda.device(self.device):
            _native.call("rtk_count_ge_f32", self.x.data_ptr(), self.n, self.m, self.ldx,
                         t.data_ptr(), counts.data_ptr(), self._stream())
        return counts.cpu().numpy()

    def launch_topk(self, k: int, search: SearchConfig, traces: bool, outputs=None, nan_word=None,
                    stream=None):
        """Enqueue the fused top-k kernel; returns (vals, idx, iters, reasons)
        device tensors (iters/reasons None without traces).  No host sync."""
        torch = _torch()
        if outputs is None:
            vals = torch.empty((self.n, k), dtype=torch.float32, device=self.device)
            idx = torch.empty((self.n, k), dtype=torch.int32, device=self.device)
            iters = torch.zeros(self.n, dtype=torch.int32, device=self.device) if traces else None
            reasons = torch.zeros(self.n, dtype=torch.int8, device=self.device) if traces else None
        else:
            vals, idx, iters, reasons = outputs
        s = self._stream() if stream is None else stream
        it_p = iters.data_ptr() if iters is not None else None
        rs_p = reasons.data_ptr() if reasons is not None else None
        nan_p = nan_word.data_ptr() if nan_word is not None else None
        ldo = int(vals.stride(0)) if self.n > 1 else int(k)
        if self.x16 is not None and not traces and (search.mode is SearchMode.EARLY_STOP or
                                                    search.epsilon_rel == 0.0):
            dtype = 1 if self.x16.dtype == torch.bfloat16 else 2
            mode = 0 if search.mode is SearchMode.EXACT else 1
            ldx16 = int(self.x16.stride(0)) if self.n > 1 else self.m
            with torch.cuda.device(self.device):
                rc = _native.load().rtk_rowtopk_x16(self.x16.data_ptr(), dtype, mode, self.n, self.m, ldx16, int(k),
                                                    int(search.hard_cap), int(search.max_iter), vals.data_ptr(),
                                                    idx.data_ptr(), ldo, nan_p, s)
            if rc != _native.RTK_EUNSUPPORTED:
                _native.check(rc, "rtk_rowtopk_x16")
                return vals, idx, iters, reasons
        with torch.cuda.device(self.device):
            if search.mode is SearchMode.EXACT:
                _native.call("rtk_rowtopk_exact_f32", self.x.data_ptr(), self.n, self.m, self.ldx, int(k),
                             float(search.epsilon_rel), int(search.hard_cap), vals.data_ptr(), idx.data_ptr(),
                             int(vals.stride(0)) if self.n > 1 else int(k), it_p, rs_p, nan_p, s)
            else:
                _native.call("rtk_rowtopk_early_f32", self.x.data_ptr(), self.n, self.m, self.ldx, int(k),
                             int(search.max_iter), vals.data_ptr(), idx.data_ptr(),
                             int(vals.stride(0)) if self.n > 1 else int(k), it_p, rs_p, nan_p, s)
        return vals, idx, iters, reasons

    def launch_trace(self, k: int, search: SearchConfig, nan_word=None):
        torch = _torch()
        iters = torch.zeros(self.n, dtype=torch.int32, device=self.device)
        reasons = torch.zeros(self.n, dtype=torch.int8, device=self.device)
        with torch.cuda.device(self.device):
            _native.call("rtk_exact_trace_f32", self.x.data_ptr(), self.n, self.m, self.ldx, int(k),
                         float(search.epsilon_rel), int(search.hard_cap), iters.data_ptr(), reasons.data_ptr(),
                         nan_word.data_ptr() if nan_word is not None else None, self._stream())
        return iters, reasons


def as_matrix(values):
    """Validate and convert to a float32 N x M matrix (batch.py:30-40).

    Host input returns a C-contiguous numpy array, CUDA input a CUDA tensor;
    the NaN scan runs on the device and names the first offending row."""
    dm = _DeviceMatrix(values)
    r = dm.first_nan_row()
    if r >= 0:
        raise NaNInputError(f"matrix contains NaN (first offending row: {r})")
    if dm.host:
        return _host_matrix(values)
    return dm.x


def resolve_workers(workers: int | str) -> int:
    """batch.py:43-49 (validated for API parity; the GPU launch ignores it)."""
    if workers == "auto":
        return max(1, os.cpu_count() or 1)
    w = int(workers)
    if w < 1:
        raise ValueError(f"workers must be >= 1 or 'auto', got {workers}")
    return w


def _workers_ok(workers) -> bool:
    try:
        resolve_workers(workers)
    except ValueError:
        return False
    return True


@dataclass(frozen=True)
class BatchConfig:
    """batch.py:52-57"""

    k: int
    search: SearchConfig = field(default_factory=SearchConfig.exact)
    workers: int | str = "auto"
    collect_traces: bool = False


@dataclass(frozen=True)
class BatchResult:
    """batch.py:60-84 -- row r of values/indices is the single-row result for row r."""

    values: object  # float32 (N, k): numpy for host input, torch.Tensor for CUDA input
    indices: object  # int32 (N, k)
    trace_iterations: object | None = None  # int32 (N,)
    trace_reasons: object | None = None  # int8 (N,)

    @property
    def n_rows(self) -> int:
        return int(self.values.shape[0])

    @property
    def k(self) -> int:
        return int(self.values.shape[1])

    def traces(self) -> list[SearchTrace]:
        if self.trace_iterations is None or self.trace_reasons is None:
            raise ValueError("traces were not collected; set collect_traces=True")
        its = self.trace_iterations.tolist()
        rs = self.trace_reasons.tolist()
        return [SearchTrace(int(i), ExitReason(int(r))) for i, r in zip(its, rs)]


def chunk_ranges(n: int, workers: int) -> list[tuple[int, int]]:
    """Contiguous near-equal [start, stop) ranges (batch.py:87-91); also the
    multi-GPU row-shard rule (shard.py)."""
    workers = min(workers, n)
    bounds = np.linspace(0, n, workers + 1, dtype=np.int64)
    return [(int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:]) if b > a]


def _to_host(t, pinned: bool = True):
    torch = _torch()
    if t is None:
        return None
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=pinned)
    h.copy_(t, non_blocking=pinned)
    return h


# Host inputs are streamed through the device in row chunks of about this
# many bytes: chunk i's H2D copy, chunk i-1's kernel and chunk i-2's D2H copy
# run concurrently (copy engines in both directions + SMs).
PIPELINE_CHUNK_BYTES = 64 << 20
PIPELINE_SLOTS = 3  # device input buffers in the chunk ring


def _launch_rows(x, k, search, vals, idx, iters, reasons, nan_word, stream):
    """One C-ABI launch over the device matrix `x` (row slices of the full
    outputs; iters/reasons may be None)."""
    n, m = int(x.shape[0]), int(x.shape[1])
    ldx = int(x.stride(0)) if n > 1 else m
    ldo = int(vals.stride(0)) if n > 1 else int(k)
    it_p = iters.data_ptr() if iters is not None else None
    rs_p = reasons.data_ptr() if reasons is not None else None
    if search.mode is SearchMode.EXACT:
        _native.call("rtk_rowtopk_exact_f32", x.data_ptr(), n, m, ldx, int(k), float(search.epsilon_rel),
                     int(search.hard_cap), vals.data_ptr(), idx.data_ptr(), ldo, it_p, rs_p,
                     nan_word.data_ptr(), stream)
    else:
        _native.call("rtk_rowtopk_early_f32", x.data_ptr(), n, m, ldx, int(k), int(search.max_iter),
                     vals.data_ptr(), idx.data_ptr(), ldo, it_p, rs_p, nan_word.data_ptr(), stream)


def _host_pipeline(xh, k: int, search: SearchConfig, traces: bool):
    """Row top-k of a host float32 matrix `xh` (CPU tensor, C-contiguous):
    chunked H2D -> kernel -> D2H on three CUDA streams, results in pinned
    host tensors.  Returns (vals, idx, iters, reasons, first_nan_row)."""
    torch = _torch()
    dev = torch.device("cuda", torch.cuda.current_device())
    n, m = int(xh.shape[0]), int(xh.shape[1])
    rows = max(1, min(n, PIPELINE_CHUNK_BYTES // (4 * m)))
    chunks = [(a, min(n, a + rows)) for a in range(0, n, rows)]
    slots = min(PIPELINE_SLOTS, len(chunks))
    pinned = xh.is_pinned()
    # pageable input: stage through pinned chunk buffers (CPU copy overlaps the GPU work)
    stage = [torch.empty((rows, m), dtype=torch.float32, pin_memory=True) for _ in range(2)] if not pinned else None
    stage_free = [None, None]
    xin = [torch.empty((rows, m), dtype=torch.float32, device=dev) for _ in range(slots)]
    vals_d = torch.empty((n, k), dtype=torch.float32, device=dev)
    idx_d = torch.empty((n, k), dtype=torch.int32, device=dev)
    it_d = torch.zeros(n, dtype=torch.int32, device=dev) if traces else None
    rs_d = torch.zeros(n, dtype=torch.int8, device=dev) if traces else None
    nan_d = torch.empty(len(chunks), dtype=torch.int32, device=dev)
    vals_h = torch.empty((n, k), dtype=torch.float32, pin_memory=True)
    idx_h = torch.empty((n, k), dtype=torch.int32, pin_memory=True)
    it_h = torch.empty(n, dtype=torch.int32, pin_memory=True) if traces else None
    rs_h = torch.empty(n, dtype=torch.int8, pin_memory=True) if traces else None
    nan_h = torch.empty(len(chunks), dtype=torch.int32, pin_memory=True)

    s_comp = torch.cuda.current_stream(dev)
    s_h2d = torch.cuda.Stream(dev)
    s_d2h = torch.cuda.Stream(dev)
    slot_free = [None] * slots  # kernel-done event of the last chunk that read each input slot
    with torch.cuda.device(dev):
        for i, (a, b) in enumerate(chunks):
            sl, r = i % slots, b - a
            src = xh[a:b]
            if not pinned:
                st = stage[i % 2]
                if stage_free[i % 2] is not None:
                    stage_free[i % 2].synchronize()  # its previous H2D has drained
                st[:r].copy_(src)
                src = st[:r]
            with torch.cuda.stream(s_h2d):
                if slot_free[sl] is not None:
                    s_h2d.wait_event(slot_free[sl])
                xin[sl][:r].copy_(src, non_blocking=True)
                h2d_done = torch.cuda.Event()
                h2d_done.record(s_h2d)
                if not pinned:
                    stage_free[i % 2] = h2d_done
            s_comp.wait_event(h2d_done)
            _launch_rows(xin[sl][:r], k, search, vals_d[a:b], idx_d[a:b],
                         it_d[a:b] if traces else None, rs_d[a:b] if traces else None,
                         nan_d[i:i + 1], s_comp.cuda_stream)
            done = torch.cuda.Event()
            done.record(s_comp)
            slot_free[sl] = done
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(done)
                vals_h[a:b].copy_(vals_d[a:b], non_blocking=True)
                idx_h[a:b].copy_(idx_d[a:b], non_blocking=True)
                if traces:
                    it_h[a:b].copy_(it_d[a:b], non_blocking=True)
                    rs_h[a:b].copy_(rs_d[a:b], non_blocking=True)
        with torch.cuda.stream(s_d2h):
            nan_h.copy_(nan_d, non_blocking=True)
        s_d2h.synchronize()
    first_nan = -1
    for i, (a, _) in enumerate(chunks):
        w = int(nan_h[i])
        if w != -1:
            first_nan = a + (w & 0xFFFFFFFF)
            break
    return vals_h, idx_h, it_h, rs_h, first_nan


def _host_tensor(matrix):
    """Host input as a C-contiguous float32 CPU tensor, validated like
    as_matrix (batch.py:30-36); pinned tensors are kept as they are."""
    torch = _torch()
    if _is_torch(matrix) and matrix.dim() == 2 and matrix.dtype == torch.float32 and not matrix.is_cuda:
        t = matrix if matrix.is_contiguous() else matrix.contiguous()
        if t.numel() == 0:
            raise EmptyRowError(f"matrix must be at least 1 x 1, got {tuple(t.shape)}")
        return t
    with warnings.catch_warnings():  # read-only arrays (memmaps) are only read from
        warnings.simplefilter("ignore", UserWarning)
        return torch.from_numpy(_host_matrix(matrix))


def batch_topk(matrix, cfg: BatchConfig) -> BatchResult:
    """Run the configured top-k search over every row (batch.py:105-142) on the
    current CUDA device.  Host inputs stream through the device in row chunks
    (H2D, kernel and D2H overlapped; results come back as numpy arrays);
    CUDA tensors are processed in place (results stay on their device)."""
    if not (_is_torch(matrix) and matrix.is_cuda):
        _require_cuda()
        xh = _host_tensor(matrix)
        k = int(cfg.k)
        m = int(xh.shape[1])
        if k < 1 or k > m or not _workers_ok(cfg.workers):
            # NaN is reported before the k-range and workers errors (batch.py:107-112)
            r = _DeviceMatrix(xh).first_nan_row()
            if r >= 0:
                raise NaNInputError(f"matrix contains NaN (first offending row: {r})")
            if k < 1 or k > m:
                raise KOutOfRangeError(f"k must be in [1, {m}], got {k}")
            resolve_workers(cfg.workers)
        vals, idx, iters, reasons, r = _host_pipeline(xh, k, cfg.search, cfg.collect_traces)
        if r >= 0:
            raise NaNInputError(f"matrix contains NaN (first offending row: {r})")
        outs = [o.numpy() if o is not None else None for o in (vals, idx, iters, reasons)]
        if cfg.collect_traces:
            return BatchResult(*outs)
        return BatchResult(outs[0], outs[1])

    dm = _DeviceMatrix(matrix)
    k = int(cfg.k)
    if k < 1 or k > dm.m or not _workers_ok(cfg.workers):
        r = dm.first_nan_row()  # NaN is reported before the k-range and workers errors (batch.py:107-112)
        if r >= 0:
            raise NaNInputError(f"matrix contains NaN (first offending row: {r})")
        if k < 1 or k > dm.m:
            raise KOutOfRangeError(f"k must be in [1, {dm.m}], got {k}")
        resolve_workers(cfg.workers)

    nan_word = dm._new_nan_word()
    vals, idx, iters, reasons = dm.launch_topk(k, cfg.search, cfg.collect_traces, nan_word=nan_word)
    r = int(nan_word.item())
    if r != -1:
        raise NaNInputError(f"matrix contains NaN (first offending row: {r & 0xFFFFFFFF})")
    if cfg.collect_traces:
        return BatchResult(vals, idx, iters, reasons)
    return BatchResult(vals, idx)


def topk_device(x, k: int, search: SearchConfig | None = None, nan_word=None):
    """Row top-k of a CUDA matrix (float32; bfloat16 / float16 rows are read
    natively where rtk_rowtopk_x16 supports the shape, others widened) enqueued on the current
    stream with no host synchronisation (capturable in a CUDA graph; the
    16-bit widening of unsupported shapes allocates): returns device
    (values, indices).  NaN rows are not raised here -- pass a 1-element
    int32 CUDA tensor as `nan_word` to receive the first offending row
    (-1 when none) and check it when convenient.  Validation of shape and k
    is done on the host as in batch_topk."""
    torch = _require_cuda()
    if not (_is_torch(x) and x.is_cuda):
        raise ValueError("topk_device expects a CUDA tensor; use batch_topk for host input")
    dm = _DeviceMatrix(x)
    k = int(k)
    if k < 1 or k > dm.m:
        raise KOutOfRangeError(f"k must be in [1, {dm.m}], got {k}")
    if nan_word is not None and (nan_word.dtype != torch.int32 or not nan_word.is_cuda or nan_word.numel() < 1):
        raise ValueError("nan_word must be a CUDA int32 tensor with at least one element")
    vals, idx, _, _ = dm.launch_topk(k, search or SearchConfig.exact(), False, nan_word=nan_word)
    return vals, idx


def exact_trace(matrix, k: int, search: SearchConfig | None = None):
    """Exit statistics only (_kernels.exact_trace_chunk, _kernels.py:217-231):
    (trace_iterations int32 (N,), trace_reasons int8 (N,))."""
    search = search or SearchConfig.exact()
    dm = _DeviceMatrix(matrix)
    if not 1 <= int(k) <= dm.m:
        raise KOutOfRangeError(f"k must be in [1, {dm.m}], got {k}")
    nan_word = dm._new_nan_word()
    iters, reasons = dm.launch_trace(int(k), search, nan_word=nan_word)
    r = int(nan_word.item())
    if r != -1:
        raise NaNInputError(f"matrix contains NaN (first offending row: {r & 0xFFFFFFFF})")
    if dm.host:
        return iters.cpu().numpy(), reasons.cpu().numpy()
    return iters, reasons
