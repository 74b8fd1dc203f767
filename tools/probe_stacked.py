"""TSQR root step at the C5 shape: P upper-triangular 8,193 x 8,193 factors (+ the tau = 1e-10
ridge), dense fls_solve of the stack vs the structure-exploiting fls_solve_stacked.

    python tools/probe_stacked.py [P ...]
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_10541_b200 import fls  # noqa: E402


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1), out


def main(Ps):
    ctx = fls.Context()
    n = 8193
    F = n - 1
    out = {}
    for P in Ps:
        lds = P * n
        g = torch.Generator(device="cuda").manual_seed(P)
        S = torch.zeros((n * lds,), dtype=torch.float64, device="cuda")
        Sv = S.view(n, lds)
        for r in range(P):
            Sv[:, r * n:(r + 1) * n] = torch.triu(torch.randn((n, n), dtype=torch.float64, device="cuda",
                                                              generator=g)).T
        sq = 1e-10 * float(torch.linalg.norm(Sv[:F]))
        fls.fls_solve_stacked(ctx, S, P, n, lds, F, sq)                 # warm-up
        ms_s, (b_s, r_s) = timed(lambda: fls.fls_solve_stacked(ctx, S, P, n, lds, F, sq))
        ld = ((lds + F + 3) // 4) * 4
        M = torch.zeros((n * ld,), dtype=torch.float64, device="cuda")
        M.view(n, ld)[:, :lds] = Sv
        ms_d, (b_d, r_d) = timed(lambda: fls.fls_solve_mu(ctx, M, lds, ld, F, sq))
        out[f"P={P}"] = {"stacked_ms": ms_s, "dense_ms": ms_d,
                         "beta_rel_diff": float(torch.linalg.norm(b_s - b_d) / torch.linalg.norm(b_d)),
                         "resid_stacked": r_s, "resid_dense": r_d}
        del S, M
        torch.cuda.empty_cache()
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [2, 4, 8])
