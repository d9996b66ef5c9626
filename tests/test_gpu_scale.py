"""GPU parity at the full BASELINE sizes:

* configs[4] (C5): N = 2^24 x M = 512, k = 64, generated on the device per
  2^20-row block (shard.device_normal_rows, the input bench.py times).  A
  sample of >= 10^4 rows spread over every block is checked bit-exactly
  against the C oracle (exact and early stop 4), and the output checksum of
  the whole matrix equals the sum of the per-shard checksums for G = 2, 4, 8
  row shards computed by the real kernel shard by shard (the multi-GPU
  partition, reference batch.py:87-102 / test_batch.py:74-81).
* configs[2] (C3) at its stated N = 2^20 for all 20 (M, k) cells, exact and
  early stop 4, on the no-trace hot path: output digests equal the
  reference's own (tests/golden/digests_c3.json, make_c3_digests.py).
* the gather path of shard.py on CUDA tensors: NCCL world size 1, and two
  ranks sharing cuda:0 over gloo, each running the real batch_topk on its
  block; the gathered result equals the unsharded launch byte for byte.
"""

import json
import os
import socket

import numpy as np
import pytest

from golden_util import GOLDEN, generate_matrix, h16

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2409_00822_b200 as rtk  # noqa: E402
from paper_2409_00822_b200.shard import (  # noqa: E402
    GEN_BLOCK_ROWS,
    device_normal_rows,
    result_checksum,
    shard_range,
    sharded_batch_topk,
)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2409_00822_b200 import _build

    _build.build()
    torch.cuda.set_device(0)


C5 = (1 << 24, 512, 64)
SEARCHES = (("exact", lambda: rtk.SearchConfig.exact()), ("early", lambda: rtk.SearchConfig.early_stop(4)))


def _u32(a):
    return np.ascontiguousarray(a).view(np.uint32)


def test_c5_sampled_rows_vs_oracle_and_shard_checksums(oracle_lib):
    n, m, k = C5
    x = device_normal_rows(m, 0, n, seed=0)
    rng = np.random.default_rng(5)
    # 768 rows from each of the 16 generator blocks, plus block edges
    rows = np.concatenate([np.sort(rng.choice(GEN_BLOCK_ROWS, 768, replace=False)) + b * GEN_BLOCK_ROWS
                           for b in range(n // GEN_BLOCK_ROWS)] +
                          [np.array([0, GEN_BLOCK_ROWS - 1, GEN_BLOCK_ROWS, n - 1])])
    rows = np.unique(rows)
    assert rows.size >= 10000
    ridx = torch.from_numpy(rows).cuda()
    sample = x.index_select(0, ridx).cpu().numpy()
    for mode, mk in SEARCHES:
        res = rtk.batch_topk(x, rtk.BatchConfig(k=k, search=mk()))
        v, i, _, _ = oracle_lib.ref_batch(sample, k, mode, max_iter=4)
        gv = res.values.index_select(0, ridx).cpu().numpy()
        gi = res.indices.index_select(0, ridx).cpu().numpy()
        assert np.array_equal(gi, i), mode
        assert np.array_equal(_u32(gv), _u32(v)), mode
        full = result_checksum(res.values, res.indices)
        del res
        # the same rows, shard by shard (each shard generated and computed on its own)
        for g in (2, 4, 8):
            total = 0
            for r in range(g):
                a, b = shard_range(n, r, g)
                xs = device_normal_rows(m, a, b, seed=0)
                assert torch.equal(xs[:4], x[a:a + 4]) and torch.equal(xs[-4:], x[b - 4:b])
                rs = rtk.batch_topk(xs, rtk.BatchConfig(k=k, search=mk()))
                total = (total + result_checksum(rs.values, rs.indices, a)) & 0xFFFFFFFFFFFFFFFF
                del xs, rs
            assert total == full, (mode, g)
    del x
    torch.cuda.empty_cache()


def _c3_cases():
    path = os.path.join(GOLDEN, "digests_c3.json")
    if not os.path.exists(path):
        return []
    with open(path) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("m", [128, 256, 512, 768, 1024])
def test_c3_full_size_reference_digests(m):
    cases = [c for c in _c3_cases() if c["M"] == m]
    assert cases, "tests/golden/digests_c3.json missing"
    x = generate_matrix(cases[0]["N"], m, 0)
    assert h16(x) == cases[0]["input"]
    xd = torch.from_numpy(x).cuda()
    del x
    for c in cases:
        search = rtk.SearchConfig.exact() if c["mode"] == "exact" else rtk.SearchConfig.early_stop(c["max_iter"])
        res = rtk.batch_topk(xd, rtk.BatchConfig(k=c["k"], search=search))  # no traces: the hot path
        assert h16(res.values.cpu().numpy(), res.indices.cpu().numpy()) == c["out"], c
    # traces for one cell per M (the general kernels' iteration / reason record)
    c = cases[0]
    search = rtk.SearchConfig.exact() if c["mode"] == "exact" else rtk.SearchConfig.early_stop(c["max_iter"])
    res = rtk.batch_topk(xd, rtk.BatchConfig(k=c["k"], search=search, collect_traces=True))
    assert h16(res.trace_iterations.cpu().numpy(), res.trace_reasons.cpu().numpy()) == c["tr"], c
    del xd, res
    torch.cuda.empty_cache()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_gather_nccl_world_one():
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        x = torch.from_numpy(generate_matrix(5000, 256, 3)).cuda()
        for _, mk in SEARCHES:
            cfg = rtk.BatchConfig(k=32, search=mk(), collect_traces=True)
            want = rtk.batch_topk(x, cfg)
            got, span = sharded_batch_topk(x, cfg, gather=True)
            assert span == (0, 5000)
            for f in ("values", "indices", "trace_iterations", "trace_reasons"):
                assert torch.equal(getattr(got, f), getattr(want, f)), f
    finally:
        dist.destroy_process_group()


def _gloo_worker(rank, world, port, n, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = torch.from_numpy(generate_matrix(n, 256, 11)).cuda()
        out = {}
        for mode, search in (("exact", rtk.SearchConfig.exact()), ("early", rtk.SearchConfig.early_stop(4))):
            cfg = rtk.BatchConfig(k=32, search=search)
            full, _ = sharded_batch_topk(x, cfg, gather=True)  # real kernel on this rank's block
            a, b = shard_range(n, rank, world)
            loc, _ = sharded_batch_topk(x[a:b].clone(), cfg, local=True, n_total=n, gather=True)
            out[mode] = (full.values.cpu().numpy(), full.indices.cpu().numpy(), loc.indices.cpu().numpy())
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_two_ranks_on_one_gpu_gather_equals_unsharded():
    import torch.multiprocessing as mp

    n, world = 3001, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    x = torch.from_numpy(generate_matrix(n, 256, 11)).cuda()
    for mode, search in (("exact", rtk.SearchConfig.exact()), ("early", rtk.SearchConfig.early_stop(4))):
        want = rtk.batch_topk(x, rtk.BatchConfig(k=32, search=search))
        wv, wi = want.values.cpu().numpy(), want.indices.cpu().numpy()
        for rank in range(world):
            fv, fi, li = got[rank][mode]
            assert np.array_equal(fi, wi) and np.array_equal(_u32(fv), _u32(wv)), (mode, rank)
            assert np.array_equal(li, wi), (mode, rank)


def test_bench_two_ranks_harness_on_one_gpu():
    """bench.py --gpus 2 end to end (self-spawn under torch.distributed.run,
    barrier + max-over-ranks timing, the C5 strong-sharded leg) with both
    ranks sharing cuda:0 over gloo (RTK_BENCH_SHARED_GPU, a harness test
    mode): one JSON line with n_gpus = 2, the C2 digests checked in the run,
    and C5 checksums equal to the 1-GPU run's (row sharding does not change
    any output)."""
    import json
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RTK_BENCH_SHARED_GPU="1")
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
                        "--no-cpu", "--no-torch", "--no-e2e", "--c5-steps", "2"],
                       capture_output=True, text=True, env=env, timeout=900, cwd=root)
    assert p.returncode == 0, p.stderr[-3000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "row shards x2 (no collective)"
    assert line["parity"]["exact"]["ok"] and line["parity"]["early"]["ok"]
    assert abs(line["value"] - 2 * (1 << 20) / (line["ms_per_step"] * 1e-3)) / line["value"] < 1e-9
    assert line["c5"]["exact"]["checksum"] == "1d0d6250a151e306"
    assert line["c5"]["early"]["checksum"] == "b601101e12c9fb17"
    assert len(line["c5"]["exact"]["per_rank_ms"]) == 2
