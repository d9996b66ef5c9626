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


def _fused_dense(x, k, search, check_nan):
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
    dense = torch.empty((n, m), dtype=x.dtype, device=x.device)
    word = torch.empty(1, dtype=torch.int32, device=x.device) if check_nan else None
    mode = 0 if search.mode is SearchMode.EXACT else 1
    with torch.cuda.device(x.device):
        rc = _native.load().rtk_maxk_dense(x.data_ptr(), _DTYPE_CODES[x.dtype], mode, n, m, ldx, int(k),
                                           int(search.hard_cap), int(search.max_iter), vals.data_ptr(),
                                           idx.data_ptr(), int(k), dense.data_ptr(), m,
                                           word.data_ptr() if word is not None else None,
                                           torch.cuda.current_stream(x.device).cuda_stream)
    if rc == _native.RTK_EUNSUPPORTED:
        return None
    _native.check(rc, "rtk_maxk_dense")
    if word is not None:
        r = int(word.item())
        if r != -1:
            raise NaNInputError(f"matrix contains NaN (first offending row: {r & 0xFFFFFFFF})")
    return dense, vals, idx


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


def to_sparse_csr(values: torch.Tensor, indices: torch.Tensor, m: int) -> torch.Tensor:
    """The fixed-k rows as a torch CSR tensor (N x m): crow = k * arange(N+1),
    col = indices (int32, ascending per row), no copy of values/indices."""
    _check_pair(values, indices)
    n, k = values.shape
    crow = torch.arange(0, n * k + 1, k, dtype=torch.int32, device=values.device)
    return torch.sparse_csr_tensor(crow, indices.contiguous().view(-1), values.contiguous().view(-1), size=(n, m))
