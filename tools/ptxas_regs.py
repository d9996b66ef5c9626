"""Registers / spills per kernel from `nvcc -Xptxas -v` output on stdin."""
import re
import sys

cur = None
for line in sys.stdin:
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = int(m.group(1)) + int(m.group(2))
        if spill:
            print(f"  SPILL {spill} bytes  {cur}")
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        print(f"{int(m.group(1)):4d} regs  {cur}")
        cur = None
