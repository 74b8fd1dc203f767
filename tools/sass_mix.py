"""Instruction mix of a SASS address range (cuobjdump -sass output), e.g. one kernel's hot loop.

    python tools/sass_mix.py file.sass 0x3100 0x3bb0
"""
import collections
import re
import sys

path, lo, hi = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
cnt = collections.Counter()
for line in open(path):
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if not m:
        continue
    addr = int(m.group(1), 16)
    if not (lo <= addr <= hi):
        continue
    toks = m.group(2).split()
    if toks and toks[0].startswith("@"):
        toks = toks[1:]
    cnt[toks[0]] += 1
for op, n in cnt.most_common():
    print(f"{n:5d} {op}")
print(f"{sum(cnt.values()):5d} total")
