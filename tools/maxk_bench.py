"""MaxK-GNN consumer kernels at the Reddit layer shape and C2: scatter (dense
MaxK output / backward of the gather) and gather (backward of MaxK), kernel
time with CUDA events vs the HBM roofline, and torch's scatter_/gather on the
same tensors.  Prints one JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_00822_b200 as rtk  # noqa: E402
from bench import peaks  # noqa: E402


def t_ms(fn, steps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    peak, _ = peaks()
    out = {"peak_GBps": peak, "cases": []}
    for n, m, k in ((232965, 256, 32), (1 << 20, 256, 32), (1 << 20, 1024, 64)):
        x = torch.randn(n, m, device="cuda")
        res = rtk.batch_topk(x, rtk.BatchConfig(k=k))
        v, i = res.values, res.indices
        il = i.long()
        dense = torch.empty(n, m, device="cuda")
        sc = t_ms(lambda: rtk.scatter_rows(v, i, m))
        ts = t_ms(lambda: dense.zero_().scatter_(1, il, v))
        ga = t_ms(lambda: rtk.gather_rows(x, i))
        tg = t_ms(lambda: torch.gather(x, 1, il))
        sb, gb = n * (4 * m + 8 * k), n * 12 * k  # algorithmic bytes: dense write + pairs read / idx+vals
        case = {"N": n, "M": m, "k": k, "scatter_ms": sc, "scatter_frac": sb / (sc * 1e-3) / 1e9 / peak,
                "torch_zero_scatter_ms": ts, "gather_ms": ga, "torch_gather_ms": tg,
                "gather_algorithmic_GBps": gb / (ga * 1e-3) / 1e9}
        if m in (128, 256):
            # MaxK forward: fused kernel vs select (topk_device) + scatter, and
            # the plain torch formulation (topk + zeros + scatter)
            for md, s in (("exact", rtk.SearchConfig.exact()), ("early", rtk.SearchConfig.early_stop(4))):
                fu = t_ms(lambda: rtk.maxk_dense_fused(x, k, s, check_nan=False))
                un = t_ms(lambda: rtk.scatter_rows(*rtk.topk_device(x, k, s), m))
                fb = n * (8 * m + 8 * k)  # read row, write dense row + values + indices
                case[f"fused_{md}_ms"] = fu
                case[f"fused_{md}_frac"] = fb / (fu * 1e-3) / 1e9 / peak
                case[f"select_scatter_{md}_ms"] = un
            case["torch_topk_scatter_ms"] = t_ms(lambda: torch.zeros_like(x).scatter_(1, *reversed(torch.topk(x, k, dim=1))), 10)
        out["cases"].append(case)
        del x, dense
        torch.cuda.empty_cache()
    # MaxK-GNN aggregation at the Reddit node count (synthetic uniform graph,
    # mean degree 50): A @ MaxK(H) over the fixed-k rows vs cuSPARSE SpMM on
    # the dense MaxK rows (torch.sparse.mm on a CSR tensor)
    n, m, k, deg = 232965, 256, 32, 50
    g = torch.Generator(device="cuda").manual_seed(0)
    h = torch.randn(n, m, device="cuda", generator=g)
    vals, idx = rtk.topk_device(h, k)
    idx8 = idx.to(torch.uint8)
    row_ptr = torch.arange(0, n * deg + 1, deg, dtype=torch.int64, device="cuda")
    col = torch.randint(0, n, (n * deg,), device="cuda", generator=g, dtype=torch.int32)
    aval = torch.rand(n * deg, device="cuda", generator=g)
    hm = rtk.scatter_rows(vals, idx, m)
    a_csr = torch.sparse_csr_tensor(row_ptr, col.to(torch.int64), aval, size=(n, n))  # one index dtype
    t_u8 = t_ms(lambda: rtk.maxk_spmm(row_ptr, col, aval, vals, idx8, m), 20)
    t_i32 = t_ms(lambda: rtk.maxk_spmm(row_ptr, col, aval, vals, idx, m), 20)
    t_cus = t_ms(lambda: torch.sparse.mm(a_csr, hm), 10)
    gt = rtk.csr_transpose(row_ptr, col, aval, n)
    gout = torch.randn(n, m, device="cuda", generator=g)
    gv = torch.empty_like(vals)
    t_bw = t_ms(lambda: rtk._native.call("rtk_maxk_spmm_backward_f32", gt[0].data_ptr(), gt[1].data_ptr(),
                                          gt[2].data_ptr(), n, gout.data_ptr(), m, idx.data_ptr(), None, k, k, m,
                                          gv.data_ptr(), torch.cuda.current_stream().cuda_stream), 10)
    nnz = n * deg
    out["aggregation"] = {"N": n, "M": m, "k": k, "mean_degree": deg, "edges": nnz,
                          "maxk_spmm_u8_ms": t_u8, "maxk_spmm_i32_ms": t_i32, "cusparse_dense_maxk_ms": t_cus,
                          "speedup_u8_vs_cusparse": t_cus / t_u8, "backward_ms": t_bw,
                          "edge_bytes_u8": nnz * (k * 5 + 8), "edge_bytes_dense": nnz * (m * 4 + 8)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
