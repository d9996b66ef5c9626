"""Small launches of every kernel family under compute-sanitizer: paired-row
(E=4, 8; masked/unmasked; odd N), long-row (E=12..32), general kernels
(traces, RegRow, GlobalRow), k == M, NaN rows, the host pipeline, the file
job, the MaxK scatter/gather, the fused MaxK rows and the aggregation.
Exits non-zero on a parity mismatch."""
import os
import sys
import tempfile

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2409_00822_b200 as rtk  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    for m in (4, 8, 100, 128, 256, 257, 384, 512, 768, 777, 1024, 1500, 2048, 2500, 3072, 4000, 4500, 6144, 8192):
        n = 67 if m <= 1024 else 19
        x = rng.standard_normal((n, m), dtype=np.float32)
        x[5] = 1.0
        x[9, : m // 2] = np.inf
        for k in sorted({1, min(33, m), m} | ({70, 150} if 512 <= m <= 1024 else set())):  # + candidate sets
            for search, mode, mi in ((rtk.SearchConfig.exact(), "exact", 4), (rtk.SearchConfig.early_stop(3), "early", 3)):
                v, i, t, r = oracle.ref_batch(x, k, mode, max_iter=mi)
                for traces in (False, True):
                    res = rtk.batch_topk(torch.from_numpy(x).cuda(), rtk.BatchConfig(k=k, search=search, collect_traces=traces))
                    assert np.array_equal(res.indices.cpu().numpy(), i), (m, k, mode, traces)
                    assert np.array_equal(res.values.cpu().numpy().view(np.uint32), v.view(np.uint32)), (m, k, mode)
        xn = x.copy()
        xn[n - 3, m - 1] = np.nan
        try:
            rtk.batch_topk(xn, rtk.BatchConfig(k=1))
            raise AssertionError("NaN not reported")
        except rtk.NaNInputError:
            pass
    for dt in (torch.bfloat16, torch.float16):  # native 16-bit rows (rtk_rowtopk_x16)
        for m in (4, 100, 128, 132, 256):
            xs = torch.randn(67, m, device="cuda").to(dt)
            x32 = xs.float().cpu().numpy()
            for search, mode, mi in ((rtk.SearchConfig.exact(), "exact", 4), (rtk.SearchConfig.early_stop(3), "early", 3)):
                v, i, _, _ = oracle.ref_batch(x32, min(7, m - 1) or 1, mode, max_iter=mi)
                res = rtk.batch_topk(xs, rtk.BatchConfig(k=min(7, m - 1) or 1, search=search))
                assert np.array_equal(res.indices.cpu().numpy(), i), (dt, m, mode)
    xd = torch.randn(1000, 256, device="cuda")
    res = rtk.batch_topk(xd, rtk.BatchConfig(k=32))
    d = rtk.scatter_rows(res.values, res.indices, 256)
    assert torch.equal(rtk.gather_rows(d, res.indices), res.values)
    # fused MaxK rows (dense + uint8 indices) and the aggregation kernels
    for dt in (torch.float32, torch.bfloat16):
        for m in (128, 256):
            xs = torch.randn(67, m, device="cuda").to(dt)
            xs[3] = 1.0
            for search in (rtk.SearchConfig.exact(), rtk.SearchConfig.early_stop(3)):
                dense, vals, idx = rtk.maxk_dense_fused(xs, 9, search)
                v8, i8 = rtk.maxk_sparse_u8(xs, 9, search)
                assert torch.equal(i8.long(), idx.long()) and torch.equal(v8, vals)
                assert torch.equal(dense, rtk.scatter_rows(vals, idx, m).to(dt))
    hv = torch.randn(300, 256, device="cuda")
    tv, ti = rtk.topk_device(hv, 40)
    rp = torch.tensor([0, 0, 3, 40, 41, 120], dtype=torch.int64, device="cuda")
    cl = torch.randint(0, 300, (120,), dtype=torch.int32, device="cuda")
    av = torch.rand(120, device="cuda")
    o1 = rtk.maxk_spmm(rp, cl, av, tv, ti, 256)
    o2 = rtk.maxk_spmm(rp, cl, av, tv, ti.to(torch.uint8), 256)
    assert torch.equal(o1, o2)
    vv = tv.clone().requires_grad_(True)
    rtk.maxk_aggregate((rp, cl, av), vv, ti, 256).sum().backward()
    with tempfile.TemporaryDirectory() as tdir:
        p, q = os.path.join(tdir, "x.rtkm"), os.path.join(tdir, "o.rtkr")
        rtk.save_matrix(rng.standard_normal((3000, 96), dtype=np.float32), p)
        rtk.topk_file(p, q, rtk.BatchConfig(k=7), chunk_rows=1000)
    print("sanitize probe ok")


if __name__ == "__main__":
    main()
