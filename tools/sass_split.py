"""Split `cuobjdump -sass` output of a .so into one file per kernel and print
instruction-mix summaries.  Usage: python tools/sass_split.py lib.so OUTDIR [regex]"""
import collections
import os
import re
import subprocess
import sys


def main():
    so, out = sys.argv[1], sys.argv[2]
    pat = re.compile(sys.argv[3]) if len(sys.argv) > 3 else None
    txt = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
    os.makedirs(out, exist_ok=True)
    cur, lines = None, []
    funcs = {}
    for ln in txt.splitlines():
        m = re.match(r"\s*Function : (\S+)", ln)
        if m:
            if cur:
                funcs[cur] = lines
            cur, lines = m.group(1), []
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if cur and m:
            lines.append(m.group(1) + " " + m.group(2).strip())
    if cur:
        funcs[cur] = lines
    for name, ls in funcs.items():
        if pat and not pat.search(name):
            continue
        with open(os.path.join(out, name[:200] + ".sass"), "w") as f:
            f.write("\n".join(ls) + "\n")
        ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", l.split(" ", 1)[1]).split(" ")[0].split(".")[0] for l in ls)
        print(name, len(ls), dict(ops.most_common(12)))


if __name__ == "__main__":
    main()
