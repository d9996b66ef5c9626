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
    print(json.dumps(out))


if __name__ == "__main__":
    main()
