"""MaxK-GNN consumer shapes around the row top-k.

MaxK-GNN (arXiv 2409.00822 applies RTop-K to it) replaces
the ReLU of a GNN layer by MaxK: every node's hidden row keeps its k largest
entries, and the aggregation SpMM consumes the result as a sparse matrix with
exactly k non-zeros per row.  The batch top-k output -- values[N,k] and
ascending int32 column indices -- is that layout already (CSR with
row_ptr[r] = k r); this module wires it into autograd and torch's sparse
formats:

  maxk(x, k)            -> (values, indices)   differentiable in values
  maxk_dense(x, k)      -> dense N x M rows with all but the top-k zeroed
                           (M = 128 / 256: one fused kernel, rtk_maxk_dense)
  scatter_rows(v, i, m) -> dense rows from (values, indices)   (rtk_scatter_rows_f32)
  gather_rows(d, i)     -> values at indices of dense rows     (rtk_gather_rows_f32)
  to_sparse_csr(v, i, m)-> torch.sparse_csr_tensor for torch.sparse.mm
  maxk_sparse_u8(x, k)  -> (values, uint8 indices)   M = 128 / 256 (fused kernel)
  maxk_aggregate(g, v, i, m) -> MaxK-GNN aggregation A @ H over the fixed-k
                           rows (rtk_maxk_spmm_f32), differentiable in v

Selection is the exact / early-stop search of batch_topk (same kernels,
bit-identical values and indices); the gradient of the selected values
w.r.t. x is the scatter of the incoming gradient to the selected columns.
All ops run on the CUDA device of their inputs; no CPU fallback.
"""

from __future__ import annotations

import torch

from . import _native
from .batch import BatchConfig, batch_topk, topk_device
from .errors import KOutOfRangeError, NaNInputError
from .select import SearchConfig, SearchMode


def _check_pair(values, indices):
    if not (values.is_cuda and indices.is_cuda):
        raise ValueError("values and indices must be CUDA tensors")
    if values.shape != indices.shape or values.dim() != 2:
        raise ValueError(f"values {tuple(values.shape)} and indices {tuple(indices.shape)} must be equal 2-D shapes")
    if indices.dtype != torch.int32:
        raise ValueError(f"indices must be int32, got {indices.dtype}")


def scatter_rows(values: torch.Tensor, indices: torch.Tensor, m: int) -> torch.Tensor:
    """out[r, indices[r, j]] = values[r, j], zeros elsewhere (N x m, float32)."""
    _check_pair(values, indices)
    v = values.to(torch.float32).contiguous()
    i = indices.contiguous()
    n, k = v.shape
    out = torch.empty((n, m), dtype=torch.float32, device=v.device)
    with torch.cuda.device(v.device):
        _native.call("rtk_scatter_rows_f32", v.data_ptr(), i.data_ptr(), k, n, k, m, out.data_ptr(), m,
                     torch.cuda.current_stream(v.device).cuda_stream)
    return out


def gather_rows(dense: torch.Tensor, indices: torch.Tensor) -> torch.Tensor:
    """values[r, j] = dense[r, indices[r, j]] (float32)."""
    if not dense.is_cuda or dense.dim() != 2:
        raise ValueError("dense must be a 2-D CUDA tensor")
    d = dense.to(torch.float32)
    if d.stride(1) != 1:
        d = d.contiguous()
    i = indices.contiguous()
    if i.dtype != torch.int32 or i.dim() != 2 or i.shape[0] != d.shape[0]:
        raise ValueError("indices must be int32 of shape (N, k)")
    n, k = i.shape
    vals = torch.empty((n, k), dtype=torch.float32, device=d.device)
    ldd = int(d.stride(0)) if n > 1 else int(d.shape[1])
    with torch.cuda.device(d.device):
        _native.call("rtk_gather_rows_f32", d.data_ptr(), ldd, i.data_ptr(), k, n, k, int(d.shape[1]),
                     vals.data_ptr(), torch.cuda.current_stream(d.device).cuda_stream)
    return vals


def _select(x, k, search, check_nan):
    if check_nan:
        res = batch_topk(x, BatchConfig(k=k, search=search))
        return res.values, res.indices
    return topk_device(x, k, search)  # no host sync: CUDA-graph capturable


class _MaxK(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, k, search, check_nan):
        values, indices = _select(x.detach(), k, search, check_nan)
        ctx.save_for_backward(indices)
        ctx.m = int(x.shape[1])
        ctx.dtype = x.dtype
        ctx.mark_non_differentiable(indices)
        return values, indices

    @staticmethod
    def backward(ctx, grad_values, _grad_indices):
        (indices,) = ctx.saved_tensors
        if grad_values is None:
            return None, None, None, None
        return scatter_rows(grad_values.contiguous(), indices, ctx.m).to(ctx.dtype), None, None, None


_DTYPE_CODES = {torch.float32: 0, torch.bfloat16: 1, torch.float16: 2}


def _fused_rows(x, k, search, check_nan, want_dense=True, want_u8=False):
    """rtk_maxk_dense: selection and dense MaxK rows from one kernel (values
    and indices as batch_topk).  None when the shape is outside its native
    path (m = 128 / 256, aligned rows) -- the caller then selects and
    scatters."""
    if not (x.is_cuda and x.dim() == 2 and x.dtype in _DTYPE_CODES and x.shape[0] > 0):
        return None
    n, m = int(x.shape[0]), int(x.shape[1])
    if m not in (128, 256) or x.stride(1) != 1:
        return None
    if search.mode is SearchMode.EXACT and search.epsilon_rel != 0.0:
        return None
    if not 1 <= k <= m:
        raise KOutOfRangeError(f"k must be in [1, {m}], got {k}")
    ldx = int(x.stride(0)) if n > 1 else m
    vals = torch.empty((n, k), dtype=torch.float32, device=x.device)
    idx = torch.empty((n, k), dtype=torch.int32, device=x.device)
    dense = torch.empty((n, m), dtype=x.dtype, device=x.device) if want_dense else None
    idx8 = torch.empty((n, k), dtype=torch.uint8, device=x.device) if want_u8 else None
    word = torch.empty(1, dtype=torch.int32, device=x.device) if check_nan else None
    mode = 0 if search.mode is SearchMode.EXACT else 1
    with torch.cuda.device(x.device):
        rc = _native.load().rtk_maxk_dense(x.data_ptr(), _DTYPE_CODES[x.dtype], mode, n, m, ldx, int(k),
                                           int(search.hard_cap), int(search.max_iter), vals.data_ptr(),
                                           idx.data_ptr(), int(k), dense.data_ptr() if dense is not None else None, m,
                                           idx8.data_ptr() if idx8 is not None else None, int(k),
                                           word.data_ptr() if word is not None else None,
                                           torch.cuda.current_stream(x.device).cuda_stream)
    if rc == _native.RTK_EUNSUPPORTED:
        return None
    _native.check(rc, "rtk_maxk_dense")
    if word is not None:
        r = int(word.item())
        if r != -1:
            raise NaNInputError(f"matrix contains NaN (first offending row: {r & 0xFFFFFFFF})")
    return dense, vals, idx, idx8


def _fused_dense(x, k, search, check_nan):
    out = _fused_rows(x, k, search, check_nan)
    return None if out is None else out[:3]


class _MaxKDense(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, k, search, check_nan):
        fused = _fused_dense(x.detach(), k, search, check_nan)
        if fused is not None:
            dense, _, indices = fused
            ctx.save_for_backward(indices)
            return dense
        values, indices = _select(x.detach(), k, search, check_nan)
        ctx.save_for_backward(indices)
        return scatter_rows(values, indices, int(x.shape[1])).to(x.dtype)  # kept values are exact in x's dtype

    @staticmethod
    def backward(ctx, grad_out):
        (indices,) = ctx.saved_tensors
        g = scatter_rows(gather_rows(grad_out, indices), indices, int(grad_out.shape[1]))
        return g.to(grad_out.dtype), None, None, None


def maxk(x: torch.Tensor, k: int, search: SearchConfig | None = None, check_nan: bool = True):
    """Row top-k of a CUDA matrix (float32, or bfloat16 / float16 read
    natively up to 4096 columns) as (float32 values, int32 indices); values carry
    the gradient (scattered back to the selected columns, in x's dtype).
    check_nan=False skips the NaN read-back (no host sync per call; the op
    can then be captured in a CUDA graph)."""
    return _MaxK.apply(x, int(k), search or SearchConfig.exact(), bool(check_nan))


def maxk_dense(x: torch.Tensor, k: int, search: SearchConfig | None = None, check_nan: bool = True) -> torch.Tensor:
    """The MaxK nonlinearity in dense form: x with all but each row's top-k
    entries set to zero, in x's dtype (gradient flows to the kept entries
    only).  Rows of 128 or 256 take the fused kernel (rtk_maxk_dense: no
    separate scatter pass); other shapes select and then scatter."""
    return _MaxKDense.apply(x, int(k), search or SearchConfig.exact(), bool(check_nan))


def maxk_dense_fused(x: torch.Tensor, k: int, search: SearchConfig | None = None, check_nan: bool = True):
    """(dense, values, indices) from the fused kernel, no autograd; raises
    ValueError when x is outside its native path (m = 128 / 256, float32 /
    bfloat16 / float16 CUDA rows with unit column stride)."""
    out = _fused_dense(x, int(k), search or SearchConfig.exact(), bool(check_nan))
    if out is None:
        raise ValueError(f"rtk_maxk_dense: unsupported input {tuple(x.shape)} {x.dtype} (stride {tuple(x.stride())})")
    return out


def maxk_sparse_u8(x: torch.Tensor, k: int, search: SearchConfig | None = None, check_nan: bool = True):
    """Row top-k as (float32 values, uint8 column indices) -- the compact
    fixed-k layout of the MaxK sparse rows for M <= 256 (5 bytes per kept
    entry instead of 8), from the fused kernel; M = 128 / 256 (else
    ValueError)."""
    out = _fused_rows(x, int(k), search or SearchConfig.exact(), bool(check_nan), want_dense=False, want_u8=True)
    if out is None:
        raise ValueError(f"rtk_maxk_dense: unsupported input {tuple(x.shape)} {x.dtype} (stride {tuple(x.stride())})")
    _, vals, _, idx8 = out
    return vals, idx8


def csr_transpose(row_ptr: torch.Tensor, col: torch.Tensor, aval: torch.Tensor | None, n_cols: int):
    """CSR of the transposed graph (row j lists the rows i with an edge
    (i, j), in ascending i; stable), for the aggregation's backward."""
    n = row_ptr.numel() - 1
    rows = torch.repeat_interleave(torch.arange(n, device=col.device, dtype=torch.int32),
                                   (row_ptr[1:] - row_ptr[:-1]).to(torch.int64))
    order = torch.sort(col.to(torch.int64), stable=True).indices
    col_t = rows[order].contiguous()
    aval_t = aval[order].contiguous() if aval is not None else None
    counts = torch.bincount(col.to(torch.int64), minlength=n_cols)
    row_ptr_t = torch.zeros(n_cols + 1, dtype=torch.int64, device=col.device)
    row_ptr_t[1:] = torch.cumsum(counts, 0)
    return row_ptr_t, col_t, aval_t


def _check_graph(row_ptr, col, aval):
    if row_ptr.dtype != torch.int64 or col.dtype != torch.int32:
        raise ValueError("graph CSR: row_ptr must be int64 and col int32")
    if aval is not None and aval.dtype != torch.float32:
        raise ValueError("graph CSR: aval must be float32 (or None for unit weights)")
    if not (row_ptr.is_cuda and col.is_cuda and (aval is None or aval.is_cuda)):
        raise ValueError("graph CSR tensors must be on the CUDA device")


def _idx_args(indices):
    if indices.dtype == torch.uint8:
        return None, indices.data_ptr()
    if indices.dtype == torch.int32:
        return indices.data_ptr(), None
    raise ValueError(f"indices must be int32 or uint8, got {indices.dtype}")


def maxk_spmm(row_ptr, col, aval, values, indices, m: int) -> torch.Tensor:
    """out[i, :] = sum over edges e = (i, j) of aval[e] * H[j, :], H the
    fixed-k rows (values at columns indices, int32 or uint8): MaxK-GNN's
    aggregation reading only the kept entries (rtk_maxk_spmm_f32).  Each
    column sums its terms in a fixed (edge) order: deterministic.  col must
    index rows of values."""
    _check_graph(row_ptr, col, aval)
    v = values.contiguous()
    i = indices.contiguous()
    if v.dtype != torch.float32 or v.shape != i.shape or v.dim() != 2:
        raise ValueError("values must be float32 and the same 2-D shape as indices")
    n_out = row_ptr.numel() - 1
    k = int(v.shape[1])
    out = torch.empty((n_out, int(m)), dtype=torch.float32, device=v.device)
    ip, i8 = _idx_args(i)
    with torch.cuda.device(v.device):
        _native.call("rtk_maxk_spmm_f32", row_ptr.data_ptr(), col.data_ptr(),
                     aval.data_ptr() if aval is not None else None, n_out, v.data_ptr(), ip, i8, k, k, int(m),
                     int(v.shape[0]), out.data_ptr(), int(m), torch.cuda.current_stream(v.device).cuda_stream)
    return out


class _MaxKAggregate(torch.autograd.Function):
    @staticmethod
    def forward(ctx, values, indices, row_ptr, col, aval, m, graph_t):
        ctx.save_for_backward(indices, row_ptr, col, aval if aval is not None else torch.empty(0))
        ctx.has_aval = aval is not None
        ctx.graph_t = graph_t
        ctx.m = int(m)
        return maxk_spmm(row_ptr, col, aval, values, indices, m)

    @staticmethod
    def backward(ctx, grad_out):
        indices, row_ptr, col, aval = ctx.saved_tensors
        aval = aval if ctx.has_aval else None
        n_in, k = indices.shape
        rpt, colt, avt = ctx.graph_t if ctx.graph_t is not None else csr_transpose(row_ptr, col, aval, n_in)
        g = grad_out.contiguous().to(torch.float32)
        gv = torch.empty((n_in, k), dtype=torch.float32, device=g.device)
        ip, i8 = _idx_args(indices.contiguous())
        with torch.cuda.device(g.device):
            _native.call("rtk_maxk_spmm_backward_f32", rpt.data_ptr(), colt.data_ptr(),
                         avt.data_ptr() if avt is not None else None, n_in, g.data_ptr(), int(g.shape[1]), ip, i8, k,
                         k, ctx.m, gv.data_ptr(), torch.cuda.current_stream(g.device).cuda_stream)
        return gv, None, None, None, None, None, None


def maxk_aggregate(graph, values, indices, m: int, graph_t=None) -> torch.Tensor:
    """MaxK-GNN aggregation A @ H with H the fixed-k rows (values, indices):
    graph = (row_ptr int64, col int32, aval float32 or None) of A; the
    gradient w.r.t. values runs over A's transpose (graph_t, computed by
    csr_transpose when not given)."""
    row_ptr, col, aval = graph
    _check_graph(row_ptr, col, aval)
    return _MaxKAggregate.apply(values, indices, row_ptr, col, aval, int(m), graph_t)


def to_sparse_csr(values: torch.Tensor, indices: torch.Tensor, m: int) -> torch.Tensor:
    """The fixed-k rows as a torch CSR tensor (N x m): crow = k * arange(N+1),
    col = indices (int32, ascending per row), no copy of values/indices."""
    _check_pair(values, indices)
    n, k = values.shape
    crow = torch.arange(0, n * k + 1, k, dtype=torch.int32, device=values.device)
    return torch.sparse_csr_tensor(crow, indices.contiguous().view(-1), values.contiguous().view(-1), size=(n, m))
