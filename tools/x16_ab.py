"""16-bit long rows, native path only (rtk_rowtopk_x16): kernel ms per shape
and mode for the library in RTK_LIBRARY.  One JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2409_00822_b200 as rtk  # noqa: E402
from tools.x16_bench import timed  # noqa: E402

out = {}
for m, k in ((384, 32), (512, 64), (640, 64)):
    x = torch.randn(1 << 20, m, device="cuda").to(torch.bfloat16)
    for mode, s in (("exact", rtk.SearchConfig.exact()), ("early", rtk.SearchConfig.early_stop(4))):
        out[f"{m}_{k}_{mode}"] = timed(lambda: rtk.topk_device(x, k, s))
print(json.dumps(out))
