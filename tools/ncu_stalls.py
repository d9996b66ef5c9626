"""Top instructions by a not-issued stall reason in an ncu source-page CSV.
Usage: python tools/ncu_stalls.py src.csv [reason=short_sb] [top=20]"""
import csv
import sys


def main():
    path = sys.argv[1]
    reason = sys.argv[2] if len(sys.argv) > 2 else "short_sb"
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    r = list(csv.reader(open(path)))
    hdr = r[1]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    ic = hdr.index(f"stall_{reason} (Not Issued)")
    rows = []
    for x in r[2:]:
        try:
            rows.append((float(x[ic] or 0), x[ia][-5:], x[isrc].strip()))
        except ValueError:
            pass
    tot = sum(v for v, _, _ in rows) or 1
    print(f"{reason}: total {tot:.0f}")
    for v, a, s in sorted(rows, reverse=True)[:top]:
        print(f"{v:6.0f} {v / tot:5.1%} {a} {s}")


if __name__ == "__main__":
    main()
