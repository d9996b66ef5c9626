"""Turn a gpu_profile_round.sh output directory into the committed profile
summaries: profiles/<tag>_ncu_<capture>.txt (key metrics, instruction mix,
stall reasons), profiles/<tag>_launches.txt (per-launch durations of the
default bench command) and profiles/ncu_traffic.json (dram bytes per launch
of the hot kernel, read by bench.py's roofline.traffic).

    python tools/ncu_to_profiles.py gpurun_out/r1c r1
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CAPTURES = {  # capture -> (bench workload key, rows)
    "c2_exact": ("c2:exact", 1 << 20),
    "c2_early": ("c2:early", 1 << 20),
    "m1024_exact": ("custom 1048576:1024:64:exact", 1 << 20),
    "m1024_early": ("custom 1048576:1024:64:early", 1 << 20),
    "m512_early": ("custom 1048576:512:64:early", 1 << 20),
    "m2048_exact": ("custom 524288:2048:64:exact", 1 << 19),
    "m2048_early": ("custom 524288:2048:64:early", 1 << 19),
    "m8192_exact": ("custom 131072:8192:128:exact", 1 << 17),
    "m512_exact": ("custom 1048576:512:64:exact", 1 << 20),
    "m128_exact": ("custom 1048576:128:32:exact", 1 << 20),
    "m128_early": ("custom 1048576:128:32:early", 1 << 20),
    "m768_exact": ("custom 1048576:768:64:exact", 1 << 20),
    "m768_early": ("custom 1048576:768:64:early", 1 << 20),
}
RAW_KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__grid_size", "launch__block_size", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
            "lts__t_bytes.sum"]


SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1.0, "us": 1e3,
         "usecond": 1e3, "msecond": 1e6, "nsecond": 1.0}


def raw_metrics(path):
    r = list(csv.reader(open(path)))
    hdr, units, vals = r[0], r[1], r[2]
    out = {}
    for key in RAW_KEYS:
        if key in hdr:
            i = hdr.index(key)
            u = units[i]
            if u in SCALE:
                base = "bytes" if "byte" in u else "ns"
                out[key] = f"{num(vals[i]) * SCALE[u]:.0f} {base}"
            else:
                out[key] = f"{vals[i]} {u}".strip()
    out["kernel"] = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    return out


def num(v):
    return float(str(v).replace(",", ""))


def main():
    src, tag = sys.argv[1], sys.argv[2]
    prof = os.path.join(ROOT, "profiles")
    traffic = {}
    tp = os.path.join(prof, "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp))
    for cap, (key, rows) in CAPTURES.items():
        rawp = os.path.join(src, f"prof_{cap}_raw.csv")
        if not os.path.exists(rawp):
            continue
        m = raw_metrics(rawp)
        dram = num(m["dram__bytes_read.sum"].split()[0]) + num(m["dram__bytes_write.sum"].split()[0])
        traffic[key] = dram
        summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), src, cap, str(rows)],
                              capture_output=True, text=True).stdout
        with open(os.path.join(prof, f"{tag}_ncu_{cap}.txt"), "w") as f:
            f.write(f"# ncu --set full --clock-control none, one launch of {m['kernel']}\n")
            f.write(f"# capture: {cap}  (python bench.py --mode ... --only-mode, see tools/gpu_profile_round.sh)\n")
            for k2 in RAW_KEYS:
                if k2 in m:
                    f.write(f"{k2:62s} {m[k2]}\n")
            f.write(f"{'dram bytes per launch (read + write)':62s} {dram:.0f}\n")
            f.write(summ)
    with open(tp, "w") as f:
        json.dump(traffic, f, indent=1, sort_keys=True)
    lp = os.path.join(src, "launches.csv")
    if os.path.exists(lp):
        text = open(lp).read()
        body = text[text.index('"ID"'):]
        r = list(csv.reader(io.StringIO(body)))
        h = r[0]
        ik, iv = h.index("Kernel Name"), h.index("Metric Value")
        agg = collections.OrderedDict()
        for row in r[1:]:
            name = re.sub(r"\(.*", "", row[ik])[:90]
            agg.setdefault(name, []).append(num(row[iv]))
        tot = sum(sum(v) for v in agg.values())
        with open(os.path.join(prof, f"{tag}_launches.txt"), "w") as f:
            f.write("# ncu --metrics gpu__time_duration.sum --clock-control none -c 80: python bench.py --steps 10 "
                    "--warmup 3 --no-cpu --no-e2e [--no-c5]\n# (cold-cache, serialised replay: compare SHARES, not absolutes)\n")
            f.write(f"{'launches':>8} {'mean us':>10} {'share':>7}  kernel\n")
            for name, v in agg.items():
                f.write(f"{len(v):8d} {sum(v) / len(v) / 1e3:10.1f} {sum(v) / tot:7.1%}  {name}\n")
    print("wrote profiles for", src)


if __name__ == "__main__":
    main()
