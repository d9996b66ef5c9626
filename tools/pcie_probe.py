"""Host<->device copy bandwidth on this box: pinned H2D, D2H, both at once,
and chunked H2D alone (what bounds batch_topk's end-to-end path)."""
import json
import time

import torch


def main():
    dev = torch.device("cuda", 0)
    n = 1 << 28  # 1 GiB of fp32
    h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    h.fill_(1.0)
    d = torch.empty(n, dtype=torch.float32, device=dev)
    o_h = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
    o_d = torch.zeros(n // 4, dtype=torch.float32, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps

    t = timed(lambda: d.copy_(h, non_blocking=True))
    res["h2d_GBps"] = n * 4 / t / 1e9
    t = timed(lambda: o_h.copy_(o_d, non_blocking=True))
    res["d2h_GBps"] = n / t / 1e9

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            o_h.copy_(o_d, non_blocking=True)

    t = timed(both)
    res["h2d_plus_d2h_ms"] = t * 1e3
    res["h2d_alone_ms"] = n * 4 / res["h2d_GBps"] / 1e6

    def chunked(c=16):
        step = n // c
        for i in range(c):
            d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)

    t = timed(chunked)
    res["h2d_chunked16_GBps"] = n * 4 / t / 1e9
    print(json.dumps(res))


if __name__ == "__main__":
    main()
