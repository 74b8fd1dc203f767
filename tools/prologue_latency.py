"""Single-thread latency (cycles) of the fused assembly prologue's pieces (csrc/bench).

    python tools/prologue_latency.py
"""
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402,F401

from paper_2602_10541_b200.build import build_microbench  # noqa: E402

lib = C.CDLL(build_microbench())
out = (C.c_longlong * 12)()
assert lib.mb_prologue_latency(out) == 0
names = ["philox_block", "feat_normal", "feat_bias", "prefactor_rec_2terms", "log_sqrt", "sincos"]
print(json.dumps({"cold_icache": dict(zip(names, list(out)[:6])),
                  "warm_icache": dict(zip(names, list(out)[6:]))}))
