"""Kernel durations of one bench step (fls_features_assemble) on a small config (torch.profiler).

    python tools/profile_small.py c2_poisson2d
"""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as wl  # noqa: E402
from paper_2602_10541_b200 import fls  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2_poisson2d"
p = wl.make_problem(name, "full")
F, R, d = p.n_features, p.n_rows, p.dim
ctx = fls.Context()
blocks = [fls.Block(torch.from_numpy(b.X).cuda(), b.terms, b.weight, torch.from_numpy(b.values).cuda(),
                    torch.from_numpy(b.fields).cuda() if b.fields is not None else None) for b in p.blocks]
bset = fls.BlockSet(blocks, d)
lda = fls.round_up(R, 4)
Ab = torch.empty(((F + 1) * lda,), dtype=torch.float64, device="cuda")
W = torch.empty((F, d), dtype=torch.float64, device="cuda")
b = torch.empty((F,), dtype=torch.float64, device="cuda")
for _ in range(5):
    fls.fls_features_assemble(ctx, d, F, p.sigma, p.seed, bset, W=W, b=b, A=Ab, lda=lda)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(20):
        fls.fls_features_assemble(ctx, d, F, p.sigma, p.seed, bset, W=W, b=b, A=Ab, lda=lda)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=8, max_name_column_width=70))
