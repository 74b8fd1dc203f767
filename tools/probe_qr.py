"""Time fls_geqrf (libfls blocked QR) vs torch.geqrf (cuSOLVER) at the solve shapes of C3, C4 and
the C5 262,144-row subset ([A | b], ridge rows included for C5), plus C2 and the paper's
Newton size (7,300 x 1,501).

    FLS_QR_NB=256 python tools/probe_qr.py [c3 c4 c5]
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_10541_b200 import fls  # noqa: E402

SHAPES = {"c2": (4800, 2001), "newton": (7300, 1501), "c3": (25000, 4001), "c4": (65000, 8001), "c5": (262144 + 8192, 8193)}


def main(names):
    ctx = fls.Context()
    out = {"nb": int(os.environ.get("FLS_QR_NB", "256")), "qr": os.environ.get("FLS_QR", "blocked")}
    for nm in names:
        m, n = SHAPES[nm]
        lda = (m + 3) // 4 * 4
        A = torch.randn((n, lda), dtype=torch.float64, device="cuda")
        M = torch.empty_like(A)
        flops = 2 * m * n * n - 2 * n ** 3 / 3
        ts = []
        for _ in range(3):
            M.copy_(A)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fls.fls_geqrf(ctx, M.view(-1), m, lda, n)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        out[nm] = {"m": m, "n": n, "ms": min(ts), "tflops": flops / min(ts) / 1e9, "all_ms": ts}
        del A, M
        torch.cuda.empty_cache()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(SHAPES))
