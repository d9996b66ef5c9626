"""Decode the Volta+ control bits of `cuobjdump -sass` output for one kernel:
stall, yield, write/read scoreboard slots, wait mask.
Usage: python tools/sass_ctrl.py lib.so kernel_substring [grep]"""
import re
import subprocess
import sys


def main():
    so, name = sys.argv[1], sys.argv[2]
    pat = sys.argv[3] if len(sys.argv) > 3 else None
    out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout.splitlines()
    on = False
    pend = None
    for ln in out:
        if "Function :" in ln:
            on = ln.split("Function :")[1].strip() == name or (name in ln and name.startswith("~") is False and ln.strip().endswith(name))
            continue
        if not on:
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4})\*/\s*(.*?);\s*/\* (0x[0-9a-f]+) \*/", ln)
        if m:
            pend = (m.group(1), m.group(2), int(m.group(3), 16))
            continue
        m2 = re.match(r"\s*/\* (0x[0-9a-f]+) \*/", ln)
        if m2 and pend:
            hi = int(m2.group(1), 16)
            ctrl = hi >> 41  # bits 105.. of the 128-bit word
            stall = ctrl & 0xF
            yld = (ctrl >> 4) & 1
            wbar = (ctrl >> 5) & 7
            rbar = (ctrl >> 8) & 7
            wmask = (ctrl >> 11) & 0x3F
            s = f"{pend[0]} st={stall:2d} y={yld} w={wbar if wbar != 7 else '-'} r={rbar if rbar != 7 else '-'} wait={wmask:06b}  {pend[1]}"
            if not pat or re.search(pat, s):
                print(s)
            pend = None


if __name__ == "__main__":
    main()
