"""One MaxK aggregation launch at the Reddit node count (for ncu)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_00822_b200 as rtk  # noqa: E402

n, m, k, deg = 232965, 256, 32, 50
g = torch.Generator(device="cuda").manual_seed(0)
h = torch.randn(n, m, device="cuda", generator=g)
vals, idx = rtk.topk_device(h, k)
idx8 = idx.to(torch.uint8)
row_ptr = torch.arange(0, n * deg + 1, deg, dtype=torch.int64, device="cuda")
col = torch.randint(0, n, (n * deg,), device="cuda", generator=g, dtype=torch.int32)
aval = torch.rand(n * deg, device="cuda", generator=g)
for _ in range(3):
    out = rtk.maxk_spmm(row_ptr, col, aval, vals, idx8, m)
torch.cuda.synchronize()
print("ok", float(out.abs().sum()))
