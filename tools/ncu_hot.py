"""Summarise an `ncu --page source --csv --print-source sass` dump: instructions
executed per row by opcode and the hottest address ranges.
Usage: python tools/ncu_hot.py dump.csv ROWS [top]"""
import collections
import csv
import re
import sys


def main():
    path, rows = sys.argv[1], float(sys.argv[2])
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
    with open(path) as f:
        r = list(csv.reader(f))
    hdr = r[1]
    ia, isrc, iex, istall = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), \
        hdr.index("Warp Stall Sampling (All Samples)")
    ops = collections.Counter()
    total = 0
    lines = []
    for row in r[2:]:
        if len(row) <= iex:
            continue
        try:
            n = float(row[iex] or 0)
            st = float(row[istall] or 0)
        except ValueError:
            continue
        src = row[isrc].strip()
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0]
        ops[op.split(".")[0]] += n
        total += n
        lines.append((row[ia], src, n, st))
    print(f"total warp-instructions per row: {total / rows:.1f}")
    for op, n in ops.most_common(25):
        print(f"  {op:12s} {n / rows:8.2f}")
    print("hottest instructions (per row, stall samples):")
    for a, s, n, st in sorted(lines, key=lambda x: -x[3])[:top]:
        print(f"  {a[-5:]} {n / rows:6.2f} {st:8.0f}  {s}")


if __name__ == "__main__":
    main()
