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
from .select import SearchConfig


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


class _MaxKDense(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, k, search, check_nan):
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
    only)."""
    return _MaxKDense.apply(x, int(k), search or SearchConfig.exact(), bool(check_nan))


def to_sparse_csr(values: torch.Tensor, indices: torch.Tensor, m: int) -> torch.Tensor:
    """The fixed-k rows as a torch CSR tensor (N x m): crow = k * arange(N+1),
    col = indices (int32, ascending per row), no copy of values/indices."""
    _check_pair(values, indices)
    n, k = values.shape
    crow = torch.arange(0, n * k + 1, k, dtype=torch.int32, device=values.device)
    return torch.sparse_csr_tensor(crow, indices.contiguous().view(-1), values.contiguous().view(-1), size=(n, m))
