"""Timings at the paper's own protocol sizes (context for BASELINE.md; the paper's problems and
GPU are unstated, so these are like-for-like in size only):

  linear  (Table 1 protocol): N = 1500 features as 3 blocks x 500 (multi-block,
          P:L85), M1 = 10,000 interior + M2 = 2,000 boundary rows, lambda = 100; 5-D Poisson
          (our C3 manufactured u*).  End to end = features + assembly + QR solve.
  newton  (Table 2 protocol): N = 1500, M1 = 5,000 interior (+ 800 BC),
          NL-Poisson -Lap u + u^3 = f, mu = 1e-10; seconds per Newton iteration.
  learnable (App. G): Helmholtz 2D, N = 500, 80 AdamW steps on sigma.

    python tools/paper_protocol.py > profiles/r01_paper_protocol.json
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import workloads as wl  # noqa: E402
from paper_2602_10541_b200 import fls  # noqa: E402
from paper_2602_10541_b200.learnable import fit_bandwidth  # noqa: E402
from paper_2602_10541_b200.newton import solve_nonlinear  # noqa: E402
from paper_2602_10541_b200.pipeline import solve_linear  # noqa: E402


def dev_blocks(p):
    return [fls.Block(torch.from_numpy(blk.X).cuda(), blk.terms, blk.weight,
                      torch.from_numpy(blk.values).cuda(),
                      torch.from_numpy(blk.fields).cuda() if blk.fields is not None else None)
            for blk in p.blocks]


def linear(ctx):
    p = wl.make_problem("c3_poisson5d", "full", n_int=10_000, per_face=200, n_features=1500)
    blocks = dev_blocks(p)
    Xt = torch.from_numpy(p.test_points(5000)).cuda()
    out = []
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sol = solve_linear(ctx, dim=5, n_features=1500, sigma=[1.0, 2.0, 3.0], seed=0,
                           blocks=blocks, block_features=[500, 500, 500])
        u = sol.evaluate(Xt)
        torch.cuda.synchronize()
        out.append(time.perf_counter() - t0)
    us = p.u_star(Xt.cpu().numpy())
    err = float(np.linalg.norm(u.cpu().numpy() - us) / np.linalg.norm(us))
    return {"rows": p.n_rows, "features": 1500, "seconds_end_to_end": min(out[1:]), "rel_l2": err,
            "paper": "0.05-0.09 s end to end on an unnamed GPU (Table 1, P:L214-218)"}


def newton(ctx):
    p = wl.make_nl_problem("nl_poisson2d", n_int=5000, per_edge=200, n_features=1500, sigma=3.0)
    W, b = p.parity_features()
    blocks = dev_blocks(p)
    Wd, bd = torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda()
    solve_nonlinear(ctx, Wd, bd, blocks[0], blocks[1:], *p.nl, max_iter=2, tol=0.0)   # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    beta, hist = solve_nonlinear(ctx, Wd, bd, blocks[0], blocks[1:], *p.nl, max_iter=10, tol=0.0)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    Xt = torch.from_numpy(p.test_points(5000)).cuda()
    u = fls.fls_eval(ctx, Wd, bd, beta, Xt).cpu().numpy()
    us = p.u_star(Xt.cpu().numpy())
    return {"rows": p.n_rows, "features": 1500, "iterations": len(hist) - 1,
            "seconds_per_iteration": dt / (len(hist) - 1),
            "rel_l2": float(np.linalg.norm(u - us) / np.linalg.norm(us)),
            "paper": "0.14-0.29 s per Newton iteration on an unnamed GPU (Table 2, P:L254-258)"}


def learnable(ctx):
    p = wl.make_helmholtz2d(n_int=3000, per_edge=200, n_features=500)
    W_hat, b = p.parity_features()
    t0 = time.perf_counter()
    L, hist = fit_bandwidth(ctx, torch.from_numpy(W_hat).cuda(), torch.from_numpy(b).cuda(),
                            dev_blocks(p), mode="scalar", init=3.0, steps=80, lr=0.3)
    torch.cuda.synchronize()
    return {"steps": 80, "sigma0": 3.0, "sigma_final": L[0][0], "loss0": hist[0]["loss"],
            "loss_final": hist[-1]["loss"], "seconds": time.perf_counter() - t0,
            "paper": "N=500, 80 AdamW steps, loss 2.1e-2 -> 8.1e-8 (App. G, P:L901-904; its own problem)"}


if __name__ == "__main__":
    ctx = fls.Context()
    print(json.dumps({"linear_table1_protocol": linear(ctx), "newton_table2_protocol": newton(ctx),
                      "learnable_bandwidth_appG": learnable(ctx)}, indent=1))
