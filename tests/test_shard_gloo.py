"""CPU, world_size 2 (gloo): the multi-GPU row-sharding logic of shard.py.

Each rank owns a contiguous row block (the reference's chunk rule,
batch.py:87-91) and computes it with no collective; the optional gather
reassembles all rows.  The per-rank compute is the injected CPU oracle here
(the worker replaces shard.batch_topk in its own process) so the
distribution plumbing is exercised without a GPU; on the GPU box the same
code calls batch_topk."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_compute(block, cfg):
    import oracle
    from paper_2409_00822_b200 import BatchResult, SearchMode

    s = cfg.search
    mode = "exact" if s.mode is SearchMode.EXACT else "early"
    v, i, t, r = oracle.ref_batch(np.asarray(block), cfg.k, mode, max_iter=s.max_iter, eps_rel=s.epsilon_rel,
                                  hard_cap=s.hard_cap, threads=1)
    if cfg.collect_traces:
        return BatchResult(v, i, t, r)
    return BatchResult(v, i)


def _worker(rank, world, port, n, m, k, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2409_00822_b200 as rtk
        from paper_2409_00822_b200 import shard
        from paper_2409_00822_b200.shard import shard_range, sharded_batch_topk

        shard.batch_topk = _oracle_compute  # test-only stand-in for the GPU kernel in this CPU worker

        x = np.random.default_rng(123).standard_normal((n, m), dtype=np.float32)
        out = {}
        for mode, search in (("exact", rtk.SearchConfig.exact()), ("early", rtk.SearchConfig.early_stop(4))):
            cfg = rtk.BatchConfig(k=k, search=search, collect_traces=True)
            local, (a, b) = sharded_batch_topk(x, cfg)
            assert (a, b) == shard_range(n, rank, world)
            full, _ = sharded_batch_topk(x, cfg, gather=True)
            blk = x[a:b]
            loc2, _ = sharded_batch_topk(blk, cfg, local=True, n_total=n, gather=True)
            out[mode] = (a, b, local.indices if local is not None else None, full.values, full.indices,
                         full.trace_iterations, full.trace_reasons, loc2.indices)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [1001, 1])
def test_two_rank_sharding_matches_single_process(n, oracle_lib):
    world, m, k = 2, 64, 9
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, m, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x = np.random.default_rng(123).standard_normal((n, m), dtype=np.float32)
    for mode in ("exact", "early"):
        v, i, t, r = oracle_lib.ref_batch(x, k, mode, max_iter=4)
        for rank in range(world):
            a, b, loc_idx, fv, fi, ft, fr, l2 = got[rank][mode]
            if b > a:
                assert np.array_equal(loc_idx, i[a:b])
            assert np.array_equal(fi, i) and np.array_equal(fv.view(np.uint32), v.view(np.uint32))
            assert np.array_equal(ft, t) and np.array_equal(fr, r)
            assert np.array_equal(l2, i)
