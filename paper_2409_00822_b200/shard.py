"""Multi-GPU row sharding: one process per GPU, no
collective on the hot path.

Rows are independent, so rank r of W owns the contiguous block
[floor(rN/W), floor((r+1)N/W)) -- the np.linspace rule of the reference's
chunk_ranges (batch.py:87-91), kept rank-aligned even when N < W -- and runs the single-GPU kernel on it.  Outputs are
byte-identical to the single-GPU result by row independence (the reference's
worker-count determinism, test_batch.py:74-81).  Gathering the blocks is
optional and off the timed path: ``gather=True`` all-gathers them through
torch.distributed (NCCL over NVLink/NVSwitch for CUDA tensors, gloo for CPU).
"""

from __future__ import annotations

import numpy as np

from .batch import BatchConfig, BatchResult, batch_topk


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """[start, stop) rows owned by `rank` (empty when n < world and rank >= n)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    bounds = np.linspace(0, n, world + 1, dtype=np.int64)
    return int(bounds[rank]), int(bounds[rank + 1])


def _dist():
    import torch.distributed as dist

    return dist


def sharded_batch_topk(matrix, cfg: BatchConfig, *, rank: int | None = None, world: int | None = None,
                       local: bool = False, n_total: int | None = None, gather: bool = False,
                       group=None) -> tuple[BatchResult, tuple[int, int]]:
    """Top-k of this rank's row block.

    matrix: all N rows (``local=False``; this rank slices its block) or just
    this rank's block (``local=True``, ``n_total`` = global N).  Returns
    (result, (start, stop)).  With ``gather=True`` the result holds all N rows
    on every rank (all_gather of padded blocks, then trimmed).  The block is
    computed by :func:`batch_topk` on this rank's current CUDA device.
    """
    dist = _dist()
    if rank is None:
        rank = dist.get_rank(group) if dist.is_initialized() else 0
    if world is None:
        world = dist.get_world_size(group) if dist.is_initialized() else 1
    if local:
        if n_total is None:
            raise ValueError("local=True needs n_total")
        a, b = shard_range(n_total, rank, world)
        if matrix.shape[0] != b - a:
            raise ValueError(f"rank {rank} block has {matrix.shape[0]} rows, expected {b - a}")
        block = matrix
    else:
        n_total = int(matrix.shape[0])
        a, b = shard_range(n_total, rank, world)
        block = matrix[a:b]
    res = batch_topk(block, cfg) if b > a else None
    if not gather:
        return res, (a, b)
    return _gather(res, cfg, n_total, world, group, block), (0, n_total)


def _gather(res, cfg, n_total, world, group, block):
    import torch

    dist = _dist()
    k = int(cfg.k)
    ranges = [shard_range(n_total, r, world) for r in range(world)]
    rows_max = max(b - a for a, b in ranges)
    on_cuda = isinstance(block, torch.Tensor) and block.is_cuda
    dev = block.device if on_cuda else torch.device("cpu")

    def to_t(x, dtype, shape):
        if x is None:
            return torch.zeros(shape, dtype=dtype, device=dev)
        t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
        return t.to(dev)

    def pad(t, rows):
        out = torch.zeros((rows_max,) + tuple(t.shape[1:]), dtype=t.dtype, device=dev)
        out[: t.shape[0]] = t
        return out

    mine = ranges[dist.get_rank(group)]
    nrows = mine[1] - mine[0]
    fields = [("values", torch.float32, (nrows, k)), ("indices", torch.int32, (nrows, k))]
    if cfg.collect_traces:
        fields += [("trace_iterations", torch.int32, (nrows,)), ("trace_reasons", torch.int8, (nrows,))]
    gathered = {}
    for name, dtype, shape in fields:
        local_t = pad(to_t(getattr(res, name) if res is not None else None, dtype, shape), rows_max)
        parts = [torch.empty_like(local_t) for _ in range(world)]
        dist.all_gather(parts, local_t, group=group)
        gathered[name] = torch.cat([p[: b - a] for p, (a, b) in zip(parts, ranges)], 0)
    if not on_cuda:
        gathered = {k_: v.numpy() for k_, v in gathered.items()}
    return BatchResult(**gathered)
