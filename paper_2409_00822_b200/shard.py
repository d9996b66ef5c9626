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


# Rows of a device-generated matrix come in fixed blocks of this many rows,
# each drawn from its own Philox stream, so a shard's rows do not depend on
# the number of shards.
GEN_BLOCK_ROWS = 1 << 20


def device_normal_rows(m: int, start: int, stop: int, seed: int = 0, device=None, out=None):
    """Rows [start, stop) of a virtual N(0,1) float32 matrix with M = m
    columns, generated on `device`: block b (rows [b*GEN_BLOCK_ROWS, ...))
    is torch.randn from a Philox generator seeded (seed * 1000003 + b).
    Identical rows whatever the sharding (the C5 input of SURVEY.md 8(d):
    2^24 x 512 is generated per shard on the device, not on the host)."""
    import torch

    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    n = stop - start
    x = out if out is not None else torch.empty((n, m), dtype=torch.float32, device=device)
    b0, b1 = start // GEN_BLOCK_ROWS, -(-stop // GEN_BLOCK_ROWS)
    for b in range(b0, b1):
        lo, hi = b * GEN_BLOCK_ROWS, (b + 1) * GEN_BLOCK_ROWS
        a, z = max(lo, start), min(hi, stop)
        g = torch.Generator(device=device).manual_seed(seed * 1000003 + b)
        if a == lo and z == hi:
            torch.randn((hi - lo, m), generator=g, device=device, dtype=torch.float32, out=x[a - start:z - start])
        else:
            blk = torch.randn((hi - lo, m), generator=g, device=device, dtype=torch.float32)
            x[a - start:z - start].copy_(blk[a - lo:z - lo])
    return x


_C1 = 0x9E3779B97F4A7C15 - (1 << 64)  # golden-ratio multiplier as a signed int64
_C2 = 0x632BE59BD9B4E019


def result_checksum(values, indices, row0: int = 0) -> int:
    """Order- and position-sensitive 64-bit checksum of a block of top-k
    rows (values as raw fp32 bits, int32 indices) starting at global row
    `row0`, computed on the tensors' device.  Checksums of row blocks add
    (mod 2^64), so the checksum of a sharded run is the sum of the shards'."""
    import torch

    n, k = int(values.shape[0]), int(values.shape[1])
    if n == 0:
        return 0
    dev = values.device
    pos = (torch.arange(n, device=dev, dtype=torch.int64).unsqueeze(1) + row0) * k + torch.arange(
        k, device=dev, dtype=torch.int64)
    w = pos * _C1 + _C2  # wraps mod 2^64 (int64 arithmetic)
    v = values.contiguous().view(torch.int32).to(torch.int64) & 0xFFFFFFFF
    i = indices.to(torch.int64)
    s = ((v * w) ^ (i * (w >> 7) + pos)).sum()
    return int(s.item()) & 0xFFFFFFFFFFFFFFFF


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
