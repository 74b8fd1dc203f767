"""Instruction mix per assembled entry of a kernel's hottest loop (the backward branch whose body
holds the most DFMA), from a built library -- a quick A/B of compile-time variants before any
GPU time is spent.

    python tools/hot_loop_mix.py libfls.so <kernel-name-substring> <entries-per-iteration>
"""
import collections
import re
import subprocess
import sys

lib, name, per = sys.argv[1], sys.argv[2], int(sys.argv[3])
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
body = next(f for f in funcs if name in f.split("\n", 1)[0])
ins = []
for line in body.splitlines():
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        toks = m.group(2).split()
        if toks and toks[0].startswith("@"):
            toks = toks[1:]
        ins.append((int(m.group(1), 16), toks[0], m.group(2)))
best = None
for i, (addr, op, txt) in enumerate(ins):
    m = re.search(r"BRA(?:\.U)? (?:!?U?P\d, )?0x([0-9a-f]+)", txt)
    if m and int(m.group(1), 16) < addr:
        lo = int(m.group(1), 16)
        seg = [o for a, o, _ in ins if lo <= a <= addr]
        if any(o.startswith("BAR") for o in seg):   # the chunk loop, not the entry loop
            continue
        nd = sum(1 for o in seg if o.startswith("DFMA"))
        if best is None or nd > best[0]:
            best = (nd, seg)
cnt = collections.Counter(best[1])
fp = sum(v for k, v in cnt.items() if k.split(".")[0] in ("DFMA", "DADD", "DMUL"))
tot = sum(cnt.values())
print(f"{tot / per:.2f} instr/entry: {fp / per:.2f} FP64 + {(tot - fp) / per:.2f} other  "
      + ", ".join(f"{k} {v}" for k, v in cnt.most_common() if k.split(".")[0] not in ("DFMA", "DADD", "DMUL")))
