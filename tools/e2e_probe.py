"""Where does batch_topk's host path spend its time?  Times the whole call
and its pieces at BASELINE C2 (2^20 x 256, k = 32) from pinned host memory."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_00822_b200 as rtk  # noqa: E402
from paper_2409_00822_b200 import batch  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def main():
    n, m, k = 1 << 20, 256, 32
    x = torch.randn((n, m), device="cuda")
    xh = x.cpu().pin_memory()
    cfg = rtk.BatchConfig(k=k, search=rtk.SearchConfig.exact())
    res = {}
    res["batch_topk_ms"] = timed(lambda: rtk.batch_topk(xh, cfg))
    for cb in (16 << 20, 32 << 20, 128 << 20, 256 << 20):
        batch.PIPELINE_CHUNK_BYTES = cb
        res[f"batch_topk_chunk{cb >> 20}MB_ms"] = timed(lambda: rtk.batch_topk(xh, cfg))
    batch.PIPELINE_CHUNK_BYTES = 64 << 20
    res["pipeline_only_ms"] = timed(lambda: batch._host_pipeline(xh, k, cfg.search, False))
    t0 = time.perf_counter()
    vh = torch.empty((n, k), dtype=torch.float32, pin_memory=True)
    res["pinned_alloc_ms"] = (time.perf_counter() - t0) * 1e3
    d = torch.empty_like(x)
    res["h2d_full_ms"] = timed(lambda: d.copy_(xh, non_blocking=True))
    res["kernel_ms"] = timed(lambda: rtk.batch_topk(x, cfg))
    print(json.dumps(res))




def hold_probe():
    n, m, k = 1 << 20, 256, 32
    x = torch.randn((n, m), device="cuda")
    xh = x.cpu().pin_memory()
    cfg = rtk.BatchConfig(k=k, search=rtk.SearchConfig.exact())
    out = {}
    for trial in ("hold", "drop"):
        res = rtk.batch_topk(xh, cfg)
        res = rtk.batch_topk(xh, cfg)
        torch.cuda.synchronize()
        ts = []
        for _ in range(6):
            if trial == "drop":
                res = None
            t0 = time.perf_counter()
            res = rtk.batch_topk(xh, cfg)
            ts.append((time.perf_counter() - t0) * 1e3)
        out[trial] = ts
    t0 = time.perf_counter()
    a = torch.empty((n, k), dtype=torch.float32, pin_memory=True)
    b = torch.empty((n, k), dtype=torch.float32, pin_memory=True)
    c = torch.empty((n, k), dtype=torch.float32, pin_memory=True)
    out["3_fresh_pinned_128MB_ms"] = (time.perf_counter() - t0) * 1e3
    print(json.dumps(out))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "hold":
        hold_probe()
    else:
        main()
