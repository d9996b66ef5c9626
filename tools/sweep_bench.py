"""BASELINE.json configs[2..4] sweep on one GPU: M x k grid at N=2^20 (exact and
early stop), the Reddit MaxK-GNN shape and the 2^24 x 512 shard config, each
with torch.topk on the same device-resident input.  Kernel time only (CUDA
events over K launches on the launching stream, inputs >> L2 except where
noted).  Writes one JSON document.

    python tools/sweep_bench.py [--out FILE] [--steps K] [--quick]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_2409_00822_b200 as rtk
    from bench import peaks

    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--shapes", default=None, help="comma list of M:k at N=2^20 (overrides the grid)")
    ap.add_argument("--no-extra", action="store_true", help="skip the Reddit and C5 shapes")
    ap.add_argument("--no-torch", action="store_true")
    args = ap.parse_args()
    peak, _ = peaks()
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream()

    def time_ms(fn, steps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    cases = []
    ms_list = [128, 256, 512, 768, 1024]
    ks = [16, 32, 64, 128]
    if args.quick:
        ms_list, ks = [256, 1024], [32, 128]
    shapes = [((1 << 20), m, k, "C3") for m in ms_list for k in ks]
    if args.shapes:
        shapes = [((1 << 20), int(t.split(":")[0]), int(t.split(":")[1]), "C3") for t in args.shapes.split(",")]
    if not args.no_extra:
        shapes.append((232965, 256, 32, "C4 Reddit (238 MB input ~ L2 size: timed back to back)"))
        shapes.append(((1 << 24), 512, 64, "C5 single-GPU share"))
    g = torch.Generator(device="cuda").manual_seed(0)
    for n, m, k, tag in shapes:
        x = torch.randn((n, m), device="cuda", generator=g)
        dm = rtk.batch._DeviceMatrix(x)
        rec = {"N": n, "M": m, "k": k, "tag": tag}
        bytes_ = n * (4 * m + 8 * k)
        steps = max(5, args.steps if n <= (1 << 20) else args.steps // 6)
        for name, search in (("exact", rtk.SearchConfig.exact()), ("early4", rtk.SearchConfig.early_stop(4))):
            outs = dm.launch_topk(k, search, False)
            ms = time_ms(lambda: dm.launch_topk(k, search, False, outputs=outs), steps)
            rec[name] = {"ms": ms, "rows_per_s": n / (ms * 1e-3), "gb_per_s": bytes_ / (ms * 1e-3) / 1e9,
                         "frac": bytes_ / (ms * 1e-3) / 1e9 / peak}
            del outs
        if n <= (1 << 20) and not args.no_torch:
            ms = time_ms(lambda: torch.topk(x, k, dim=1, sorted=True), max(3, steps // 5))
            rec["torch_topk_sorted"] = {"ms": ms, "rows_per_s": n / (ms * 1e-3)}
            rec["speedup_exact"] = ms / rec["exact"]["ms"]
            rec["speedup_early4"] = ms / rec["early4"]["ms"]
        cases.append(rec)
        print(json.dumps(rec), flush=True)
        del x, dm
        torch.cuda.empty_cache()
    doc = {"peak_gbs": peak, "gpu": torch.cuda.get_device_name(0), "cases": cases}
    if args.out:
        with open(args.out, "w") as f:
            json.dump(doc, f, indent=1)


if __name__ == "__main__":
    main()
