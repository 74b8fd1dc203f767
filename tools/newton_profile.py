"""Where one Newton iteration spends its time (Table 2 protocol size: N = 1500, M1 = 5000):
wall time of each libfls call of solve_nonlinear's loop, synchronised per call.

    python tools/newton_profile.py
"""
import json
import os
import sys
import time
from collections import defaultdict

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as wl  # noqa: E402
from paper_2602_10541_b200 import fls  # noqa: E402
from paper_2602_10541_b200 import newton  # noqa: E402

T = defaultdict(float)
N = defaultdict(int)


def wrap(name, fn):
    def f(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        T[name] += time.perf_counter() - t0
        N[name] += 1
        return r
    return f


def main():
    p = wl.make_nl_problem("nl_poisson2d", n_int=5000, per_edge=200, n_features=1500)
    W, b = p.parity_features()
    ctx = fls.Context()
    blocks = [fls.Block(torch.from_numpy(blk.X).cuda(), blk.terms, blk.weight,
                        torch.from_numpy(blk.values).cuda()) for blk in p.blocks]
    Wd, bd = torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda()
    newton.solve_nonlinear(ctx, Wd, bd, blocks[0], blocks[1:], *p.nl, max_iter=2, tol=0.0)
    for nm in ["fls_eval", "fls_nl_residual", "fls_assemble", "fls_solve_mu", "fls_axpy"]:
        setattr(newton.fls, nm, wrap(nm, getattr(fls, nm)))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, hist = newton.solve_nonlinear(ctx, Wd, bd, blocks[0], blocks[1:], *p.nl, max_iter=10, tol=0.0)
    total = time.perf_counter() - t0
    its = len(hist) - 1
    print(json.dumps({"iterations": its, "s_per_iteration": total / its,
                      "per_iteration_ms": {k: 1e3 * v / its for k, v in T.items()},
                      "calls_per_iteration": {k: v / its for k, v in N.items()}}, indent=1))


if __name__ == "__main__":
    main()
