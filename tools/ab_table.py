"""Summarise a tools/gpu_shapes_exact.sh run: ms per step of each library
variant per shape, and the ratio of the second to the first.

    python tools/ab_table.py gpurun_out/TAG base rot
"""
import collections
import glob
import json
import os
import sys

d, a, b = sys.argv[1], sys.argv[2], sys.argv[3]
r = collections.defaultdict(dict)
for f in sorted(glob.glob(os.path.join(d, "b_*.json"))):
    name = os.path.basename(f)[2:-5]
    try:
        line = json.loads(open(f).read().strip().splitlines()[-1])
    except (ValueError, IndexError):
        print(name, "no bench line")
        continue
    for lib in (a, b):
        if name.startswith(lib + "_"):
            r[name[len(lib) + 1:]][lib] = (line["ms_per_step"], line["roofline"]["frac"])
for shape, v in sorted(r.items()):
    if len(v) == 2:
        print(f"{shape:28s} {a} {v[a][0]:.4f} {b} {v[b][0]:.4f} ratio {v[b][0] / v[a][0]:.3f} frac {v[b][1]:.3f}")
