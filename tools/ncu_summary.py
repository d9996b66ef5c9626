"""One-screen summary of a gpu_ncu_variant.sh export: duration, issue, IPC,
stall reasons (not-issued), per-row instruction mix.
Usage: python tools/ncu_summary.py DIR MODE [rows]"""
import collections
import csv
import re
import sys


def main():
    d, mode = sys.argv[1], sys.argv[2]
    rows = float(sys.argv[3]) if len(sys.argv) > 3 else float(1 << 20)
    det = open(f"{d}/prof_{mode}_details.txt").read()
    print(f"  capture {mode}: {rows:.0f} rows")
    for key in ("Duration", "DRAM Throughput", "Issue Slots Busy", "Executed Ipc Active", "Registers Per Thread",
                "Achieved Occupancy", "No Eligible", "Eligible Warps Per Scheduler"):
        m = re.search(rf"^\s*{re.escape(key)}\s+(\S+)\s+(\S+)", det, re.M)
        if m:
            print(f"  {key:32s} {m.group(2)} {m.group(1)}")
    r = list(csv.reader(open(f"{d}/prof_{mode}_src.csv")))
    hdr = r[1]
    iex, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
    stall = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" in h]
    ops, st = collections.Counter(), collections.Counter()
    tot = 0.0
    for x in r[2:]:
        try:
            e = float(x[iex] or 0) / rows
        except ValueError:
            continue
        tot += e
        ops[x[isrc].split()[0] if not x[isrc].strip().startswith("@") else x[isrc].split()[1]] += e
        for i, h in stall:
            try:
                st[h.split(" ")[0]] += float(x[i] or 0)
            except ValueError:
                pass
    s = sum(st.values()) or 1
    print(f"  warp-instructions per row: {tot:.1f}")
    print("  not-issued stalls: " + ", ".join(f"{k[6:]} {v / s:.0%}" for k, v in st.most_common(6)))
    print("  mix: " + ", ".join(f"{k.split('.')[0]} {v:.1f}" for k, v in ops.most_common(18)))


if __name__ == "__main__":
    main()
