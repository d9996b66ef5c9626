"""16-bit input rows at C2 (2^20 x 256, k = 32): native bf16 / fp16 reads
(rtk_rowtopk_x16) vs widening to float32 first (x.float() + the fp32
kernel) vs float32 input.  Device-resident inputs (> L2), CUDA events, one
JSON line per case.  Roofline bytes: N (2 M + 8 k) for 16-bit input."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_00822_b200 as rtk  # noqa: E402

PEAK = 6558.7


def timed(fn, steps=50, warmup=5):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


def main():
    for m, k in ((256, 32), (512, 64), (1024, 64), (2048, 64)):
        run(1 << 20, m, k)


def run(n, m, k):
    x32 = torch.randn(n, m, device="cuda")
    for mode, search in (("exact", rtk.SearchConfig.exact()), ("early4", rtk.SearchConfig.early_stop(4))):
        for name, dt in (("bf16", torch.bfloat16), ("fp16", torch.float16)):
            x = x32.to(dt)
            nat = timed(lambda: rtk.topk_device(x, k, search))
            wid = timed(lambda: rtk.topk_device(x.float(), k, search))
            gb = n * (2 * m + 8 * k) / 1e9
            print(json.dumps({"M": m, "k": k, "input": name, "mode": mode, "native_ms": nat, "widen_then_f32_ms": wid,
                              "speedup": wid / nat, "native_gbs": gb / nat * 1e3,
                              "native_frac": gb / nat * 1e3 / PEAK}))
        f = timed(lambda: rtk.topk_device(x32, k, search))
        print(json.dumps({"M": m, "k": k, "input": "f32", "mode": mode, "ms": f, "frac": n * (4 * m + 8 * k) / 1e9 / f * 1e3 / PEAK}))


if __name__ == "__main__":
    main()
