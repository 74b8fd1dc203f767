"""Run a few fls_features_assemble steps of one config (target for ncu captures).

    python tools/one_step.py c2_poisson2d [steps]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as wl  # noqa: E402
from paper_2602_10541_b200 import fls  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2_poisson2d"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
p = wl.make_problem(name, "full")
F, R, d = p.n_features, p.n_rows, p.dim
ctx = fls.Context()
bset = fls.BlockSet([fls.Block(torch.from_numpy(b.X).cuda(), b.terms, b.weight, torch.from_numpy(b.values).cuda(),
                               torch.from_numpy(b.fields).cuda() if b.fields is not None else None)
                     for b in p.blocks], d)
lda = fls.round_up(R, 4)
Ab = torch.empty(((F + 1) * lda,), dtype=torch.float64, device="cuda")
W = torch.empty((F, d), dtype=torch.float64, device="cuda")
b = torch.empty((F,), dtype=torch.float64, device="cuda")
for _ in range(steps):
    fls.fls_features_assemble(ctx, d, F, p.sigma, p.seed, bset, W=W, b=b, A=Ab, lda=lda)
fls.fls_sync(ctx)
print("ok", name, steps)
