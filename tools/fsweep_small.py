"""Step time of a small config against the feature count (fixed rows): the intercept is the
per-launch fixed cost, the slope the per-feature cost (tools/small_step_probe.py's graph step).

    python tools/fsweep_small.py c2_poisson2d 250 500 1000 2000 4000
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import workloads as wl  # noqa: E402
from paper_2602_10541_b200 import fls  # noqa: E402
from small_step_probe import graph_us  # noqa: E402

name = sys.argv[1]
s = torch.cuda.Stream()
for F in [int(v) for v in sys.argv[2:]]:
    p = wl.make_problem(name, "full", n_features=F)
    R, d = p.n_rows, p.dim
    ctx = fls.Context(stream=s)
    bset = fls.BlockSet([fls.Block(torch.from_numpy(b.X).cuda(), b.terms, b.weight,
                                   torch.from_numpy(b.values).cuda(),
                                   torch.from_numpy(b.fields).cuda() if b.fields is not None else None)
                         for b in p.blocks], d)
    lda = fls.round_up(R, 4)
    Ab = torch.empty(((F + 1) * lda,), dtype=torch.float64, device="cuda")
    W = torch.empty((F, d), dtype=torch.float64, device="cuda")
    b = torch.empty((F,), dtype=torch.float64, device="cuda")
    fused = lambda: fls.fls_features_assemble(ctx, d, F, p.sigma, p.seed, bset, W=W, b=b, A=Ab, lda=lda)
    t = graph_us(fused, s, per_graph=10)
    print(json.dumps({"config": name, "F": F, "rows": R, "graph10_us": round(t, 2),
                      "entries_per_us": round(R * F / t, 1)}), flush=True)
