"""Newton-Raphson for nonlinear PDEs  L[u] + N(u, Du) = f  (Eq. 4-5) on the device.

Host orchestration only; every arithmetic step is a libfls call:
  u, L[u_N], D^e u_N at the points      fls_eval (identity / operator; A never materialised)
  -R and the N' fields                  fls_nl_residual / fls_nl_residual2
  J = [L + N_u I + N_Du D^e ; lam I]    fls_assemble (each N' term is one coefficient field)
  delta = argmin |J d + R|^2 + mu |d|^2 fls_solve_mu (Householder QR with sqrt(mu) I rows)
  beta + alpha delta                    fls_axpy
Warm start from the linear part, Armijo backtracking on the residual norm, stop on
||du|| / ||u|| at the collocation points, and continuation (homotopy) over a parameter
schedule for advection-dominated problems (readings N1-N5 in DESIGN.md §3).

Nonlinearities: ('poly', [a0, a1, ...]) = sum_k a_k u^k; ('exp', [a0, a1]) = a0 exp(a1 u);
('udu', [a0], alpha) = a0 u D^alpha u (steady Burgers u u_x with alpha = e_x).
"""
from __future__ import annotations

import math
from typing import Callable, List, Optional, Sequence

import torch

from . import fls


def solve_nonlinear(ctx: fls.Context, W: torch.Tensor, b: torch.Tensor, pde: fls.Block,
                    bcs: Sequence[fls.Block], nl_kind: str, nl_coefs: Sequence[float],
                    nl_alpha: Optional[Sequence[int]] = None, *, mu: float = 1e-10,
                    max_iter: int = 30, tol: float = 1e-10, c_armijo: float = 1e-4,
                    max_halvings: int = 30, beta0: Optional[torch.Tensor] = None):
    """Returns (beta, history).  pde.values = f, bc.values = g; pde.terms = L (constant
    coefficients); bc blocks carry their operator B in bc.terms (identity for Dirichlet rows;
    Neumann / Robin with constant coefficients), used by both the residual and the Jacobian.
    beta0: start from these coefficients instead of the linear warm start (continuation).
    history entries: resid, alpha (the step actually taken), du_rel, armijo (False when the
    line search exhausted max_halvings and took its last, non-decreasing trial)."""
    F, d = int(W.shape[0]), int(W.shape[1])
    nl = fls.make_nonlinearity(nl_kind, nl_coefs)
    quasi = nl_kind == "udu"
    if quasi and nl_alpha is None:
        raise ValueError("'udu' needs nl_alpha (the derivative D^alpha in a0 u D^alpha u)")
    d_terms = [(tuple(nl_alpha), 1.0, -1)] if quasi else None
    zero_nl = fls.make_nonlinearity("poly", [0.0])
    bc_identity = [len(bc.terms) == 1 and not any(bc.terms[0][0]) and bc.terms[0][1] == 1.0
                   and bc.terms[0][2] == -1 for bc in bcs]
    for bc in bcs:
        if any(int(t[2]) >= 0 for t in bc.terms):
            raise ValueError("BC operators with coefficient fields are not supported (fls_eval)")
    sq = math.sqrt(mu)
    R = pde.n + sum(bc.n for bc in bcs)
    lda = fls.round_up(R + F, 4)
    Ab = torch.empty(((F + 1) * lda,), dtype=torch.float64, device=W.device)
    if beta0 is None:
        # warm start: the linear part (N dropped), one Tikhonov-regularised solve
        fls.fls_assemble(ctx, W, b, [pde] + list(bcs), A=Ab, lda=lda)
        beta, _ = fls.fls_solve_mu(ctx, Ab, R, lda, F, sq)
    else:
        beta = beta0.clone()
    zero = tuple([0] * d)

    def state(beta, u_prev=None):
        u = fls.fls_eval(ctx, W, b, beta, pde.X)
        Lu = fls.fls_eval(ctx, W, b, beta, pde.X, terms=pde.terms)
        if quasi:
            Du = fls.fls_eval(ctx, W, b, beta, pde.X, terms=d_terms)
            neg, dN, dN2, st = fls.fls_nl_residual2(ctx, nl, Lu, u, Du, pde.values, u_prev=u_prev)
            fields = [dN, dN2]
        else:
            neg, dN, st = fls.fls_nl_residual(ctx, nl, Lu, u, pde.values, u_prev=u_prev)
            fields = [dN]
        r2 = st[0]
        negs = [neg]
        for bc, ident in zip(bcs, bc_identity):
            # B[u](x_b): the BC operator itself (the same rows the Jacobian assembles)
            ub = fls.fls_eval(ctx, W, b, beta, bc.X, terms=None if ident else bc.terms)
            nb, _, stb = fls.fls_nl_residual(ctx, zero_nl, ub, ub, bc.values)
            negs.append(nb)
            r2 += bc.weight ** 2 * stb[0]
        return u, fields, negs, math.sqrt(r2), st

    u, fields, negs, rn, _ = state(beta)
    hist: List[dict] = [{"resid": rn, "alpha": None, "du_rel": None}]
    for _ in range(max_iter):
        base = 0 if pde.fields is None else int(pde.fields.shape[1])
        cols = ([pde.fields] if pde.fields is not None else []) + [f.view(-1, 1) for f in fields]
        jac_terms = list(pde.terms) + [(zero, 1.0, base)]
        if quasi:
            jac_terms.append((tuple(nl_alpha), 1.0, base + 1))
        J = [fls.Block(pde.X, jac_terms, 1.0, negs[0], torch.cat(cols, 1).contiguous())]
        J += [fls.Block(bc.X, bc.terms, bc.weight, nb) for bc, nb in zip(bcs, negs[1:])]
        fls.fls_assemble(ctx, W, b, J, A=Ab, lda=lda)
        delta, _ = fls.fls_solve_mu(ctx, Ab, R, lda, F, sq)
        alpha, armijo = 1.0, False
        for _h in range(max(1, max_halvings)):
            trial = fls.fls_axpy(ctx, alpha, delta, beta)
            u_t, fields_t, negs_t, rn_t, st_t = state(trial, u_prev=u)
            if rn_t <= (1.0 - c_armijo * alpha) * rn:
                armijo = True
                break
            if _h + 1 < max_halvings:
                alpha *= 0.5
        du = math.sqrt(st_t[2]) / max(math.sqrt(st_t[1]), 1e-300)
        beta, u, fields, negs, rn = trial, u_t, fields_t, negs_t, rn_t
        hist.append({"resid": rn, "alpha": alpha, "du_rel": du, "armijo": armijo})
        if du < tol:
            break
    return beta, hist


def solve_continuation(ctx: fls.Context, W: torch.Tensor, b: torch.Tensor,
                       make_pde: Callable[[float], fls.Block], bcs: Sequence[fls.Block],
                       nl_kind: str, nl_coefs: Sequence[float], schedule: Sequence[float],
                       nl_alpha: Optional[Sequence[int]] = None, **kw):
    """Continuation / homotopy: solve along the parameter schedule (e.g. viscosity
    1.0 -> 0.5 -> 0.2 -> 0.1), each stage warm-started from the previous stage's beta.
    Returns (beta, [history per stage])."""
    beta, hists = None, []
    for p in schedule:
        beta, h = solve_nonlinear(ctx, W, b, make_pde(p), bcs, nl_kind, nl_coefs, nl_alpha,
                                  beta0=beta, **kw)
        hists.append(h)
    return beta, hists
