"""Registers / spills per kernel from the build's ptxas -v logs.

    python tools/ptxas_table.py [build_dir] [name-filter]
"""
import glob
import os
import re
import sys

d = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "..", "paper_2602_10541_b200", "_build")
flt = sys.argv[2] if len(sys.argv) > 2 else ""
for f in sorted(glob.glob(os.path.join(d, "*.ptxas.txt"))):
    cur = None
    for line in open(f):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = m.group(1)
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m and cur:
            st = m.groups()
        m = re.search(r"Used (\d+) registers", line)
        if m and cur and flt in cur:
            print(f"{cur:70s} regs {m.group(1):>3s} stack {st[0]:>4s} spill {st[1]}/{st[2]}")
            cur = None
