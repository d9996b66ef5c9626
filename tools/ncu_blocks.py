"""Basic blocks of an `ncu --page source --csv --print-source sass` dump:
consecutive instructions with the same execution count, with instructions
per row (count x length / rows).  Usage: python tools/ncu_blocks.py src.csv ROWS [min_per_row]"""
import csv
import sys


def main():
    path, rows = sys.argv[1], float(sys.argv[2])
    lim = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
    r = list(csv.reader(open(path)))
    h = r[1]
    ia, isrc, ie = h.index("Address"), h.index("Source"), h.index("Instructions Executed")
    blocks, cur = [], None
    for x in r[2:]:
        try:
            n = float(x[ie] or 0)
        except ValueError:
            continue
        if cur and cur[2] == n:
            cur[1] = x[ia]
            cur[3] += 1
            cur[4].append(x[isrc].strip().split(" ")[0])
        else:
            cur = [x[ia], x[ia], n, 1, [x[isrc].strip().split(" ")[0]]]
            blocks.append(cur)
    tot = sum(b[2] * b[3] for b in blocks) / rows
    print(f"total per row {tot:.1f}")
    for a0, a1, n, ln, ops in blocks:
        pr = n * ln / rows
        if pr >= lim:
            print(f"{a0[-5:]}-{a1[-5:]} x{n / rows:6.3f} len {ln:3d} -> {pr:6.1f}/row  {' '.join(o for o in ops[:6])} ...")


if __name__ == "__main__":
    main()
