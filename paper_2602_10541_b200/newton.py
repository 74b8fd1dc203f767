"""Newton-Raphson for nonlinear PDEs  L[u] + N(u) = f  (Eq. 4-5) on the device.

Host orchestration only; every arithmetic step is a libfls call:
  u, L[u_N] at the collocation points   fls_eval (identity / operator; A never materialised)
  -R and N'(u)                          fls_nl_residual (pointwise N, deterministic norms)
  J = [L + N'(u) I ; lam I] rows        fls_assemble (the N' term is one coefficient field)
  delta = argmin |J d + R|^2 + mu |d|^2 fls_solve (Householder QR with sqrt(mu) I rows)
  beta + alpha delta                    fls_axpy
Warm start from the linear part, Armijo backtracking on the residual norm, stop on
||du|| / ||u|| at the collocation points (readings N1-N5 in DESIGN.md §3).
"""
from __future__ import annotations

import math
from typing import List, Sequence

import torch

from . import fls


def solve_nonlinear(ctx: fls.Context, W: torch.Tensor, b: torch.Tensor, pde: fls.Block,
                    bcs: Sequence[fls.Block], nl_kind: str, nl_coefs: Sequence[float], *,
                    mu: float = 1e-10, max_iter: int = 30, tol: float = 1e-10,
                    c_armijo: float = 1e-4, max_halvings: int = 30):
    """Returns (beta, history).  pde.values = f, bc.values = g; pde.terms = L (constant
    coefficients); every bc block's operator is evaluated as the identity (Dirichlet rows)."""
    F, d = int(W.shape[0]), int(W.shape[1])
    nl = fls.make_nonlinearity(nl_kind, nl_coefs)
    zero_nl = fls.make_nonlinearity("poly", [0.0])
    sq = math.sqrt(mu)
    R = pde.n + sum(bc.n for bc in bcs)
    lda = fls.round_up(R + F, 4)
    Ab = torch.empty(((F + 1) * lda,), dtype=torch.float64, device=W.device)
    # warm start: the linear part (N dropped), one Tikhonov-regularised solve
    fls.fls_assemble(ctx, W, b, [pde] + list(bcs), A=Ab, lda=lda)
    beta, _ = fls.fls_solve(ctx, Ab, R, lda, F, sq)
    zero = tuple([0] * d)

    def state(beta, u_prev=None):
        u = fls.fls_eval(ctx, W, b, beta, pde.X)
        Lu = fls.fls_eval(ctx, W, b, beta, pde.X, terms=pde.terms)
        neg, dN, st = fls.fls_nl_residual(ctx, nl, Lu, u, pde.values, u_prev=u_prev)
        r2 = st[0]
        negs = [neg]
        for bc in bcs:
            ub = fls.fls_eval(ctx, W, b, beta, bc.X)
            nb, _, stb = fls.fls_nl_residual(ctx, zero_nl, ub, ub, bc.values)
            negs.append(nb)
            r2 += bc.weight ** 2 * stb[0]
        return u, dN, negs, math.sqrt(r2), st

    u, dN, negs, rn, _ = state(beta)
    hist: List[dict] = [{"resid": rn, "alpha": None, "du_rel": None}]
    for _ in range(max_iter):
        fields = dN.view(-1, 1) if pde.fields is None else torch.cat([pde.fields, dN.view(-1, 1)], 1)
        gid = 0 if pde.fields is None else int(pde.fields.shape[1])
        J = [fls.Block(pde.X, list(pde.terms) + [(zero, 1.0, gid)], 1.0, negs[0], fields.contiguous())]
        J += [fls.Block(bc.X, bc.terms, bc.weight, nb) for bc, nb in zip(bcs, negs[1:])]
        fls.fls_assemble(ctx, W, b, J, A=Ab, lda=lda)
        delta, _ = fls.fls_solve(ctx, Ab, R, lda, F, sq)
        alpha = 1.0
        for _h in range(max_halvings):
            trial = fls.fls_axpy(ctx, alpha, delta, beta)
            u_t, dN_t, negs_t, rn_t, st_t = state(trial, u_prev=u)
            if rn_t <= (1.0 - c_armijo * alpha) * rn:
                break
            alpha *= 0.5
        du = math.sqrt(st_t[2]) / max(math.sqrt(st_t[1]), 1e-300)
        beta, u, dN, negs, rn = trial, u_t, dN_t, negs_t, rn_t
        hist.append({"resid": rn, "alpha": alpha, "du_rel": du})
        if du < tol:
            break
    return beta, hist
