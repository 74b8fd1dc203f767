"""Kernel-time breakdown of one fls_geqrf call (torch.profiler / CUPTI; no nsys on the box).

    python tools/profile_qr.py c3
"""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_10541_b200 import fls  # noqa: E402
from tools.probe_qr import SHAPES  # noqa: E402

nm = sys.argv[1] if len(sys.argv) > 1 else "c3"
m, n = SHAPES[nm]
lda = (m + 3) // 4 * 4
ctx = fls.Context()
A = torch.randn((n, lda), dtype=torch.float64, device="cuda")
M = A.clone()
fls.fls_geqrf(ctx, M.view(-1), m, lda, n)
M.copy_(A)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    fls.fls_geqrf(ctx, M.view(-1), m, lda, n)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=90))
