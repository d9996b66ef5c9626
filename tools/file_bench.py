"""File-level job throughput: a BASELINE C2-shaped RTKM file (2^20 x 256 fp32,
1 GiB) -> topk_file (native streaming pipeline) -> RTKR, versus the
reference-style chain load_matrix -> batch_topk -> save_result on the same
GPU.  The file is written once and read from the page cache; times are wall
clock of the whole job (median of runs).  Prints one JSON line."""
import json
import os
import statistics
import sys
import tempfile
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_00822_b200 as rtk  # noqa: E402


def main():
    n, m, k = 1 << 20, 256, 32
    base = sys.argv[1] if len(sys.argv) > 1 else None
    d = tempfile.mkdtemp(prefix="rtk_file_", dir=base)
    src, out, out2 = (os.path.join(d, f) for f in ("x.rtkm", "o.rtkr", "o2.rtkr"))
    x = np.random.default_rng(0).standard_normal((n, m), dtype=np.float32)
    rtk.save_matrix(x, src)
    cfg = rtk.BatchConfig(k=k)
    res = {"workload": "RTKM 2^20 x 256 fp32 (1 GiB, page cache) -> RTKR k=32, exact", "dir": d}
    rtk.topk_file(src, out, cfg)  # warm-up (page cache, allocations)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        rtk.topk_file(src, out, cfg)
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    res["topk_file_ms"] = t * 1e3
    res["topk_file_rows_per_s"] = n / t
    res["topk_file_input_GBps"] = n * m * 4 / t / 1e9
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        rtk.save_result(rtk.batch_topk(rtk.load_matrix(src), cfg), out2)
        ts.append(time.perf_counter() - t0)
    t2 = statistics.median(ts)
    res["chain_load_batch_save_ms"] = t2 * 1e3
    res["identical_bytes"] = open(out, "rb").read() == open(out2, "rb").read()
    for f in (src, out, out2):
        os.unlink(f)
    os.rmdir(d)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
