"""Oracle Newton-Raphson for L[u] + N(u) = f (Eq. 4-5) -- TEST INFRASTRUCTURE ONLY.

Step by step in the paper's order (readings N1-N5 in DESIGN.md §3):
  warm start  : beta_0 = Tikhonov lstsq of the linear part (N dropped)
  residual    : R = [(L + N)[u_N](x_i) - f_i ; lam (u_N(x_b) - g_b)]
  Jacobian    : J = [L[phi_j](x_i) + N'(u_i) s phi_j(x_i) ; lam s phi_j(x_b)]
  step        : delta = argmin ||J delta + R||^2 + mu ||delta||^2, mu = 1e-10
  line search : alpha = 1, halve while ||R(beta + alpha delta)|| > (1 - c alpha)||R(beta)||,
                c = 1e-4 (Armijo sufficient decrease on the residual norm)
  stop        : ||u_{k+1} - u_k|| / ||u_{k+1}|| < tol at the collocation points
Primitives: orc_assemble (term-by-term closed form), orc_lstsq_mu (Householder QR),
orc_eval, numpy matrix-vector products and the pointwise N, N'.
"""
from __future__ import annotations

import math

import numpy as np

from . import assemble, evaluate, lstsq_mu


def nl_funcs(kind, coefs):
    c = list(coefs)
    if kind == "poly":
        def N(u):
            return np.zeros_like(u) + sum(ck * u ** k for k, ck in enumerate(c))

        def dN(u):
            return np.zeros_like(u) + sum(k * ck * u ** (k - 1) for k, ck in enumerate(c) if k > 0)
    elif kind == "exp":
        def N(u):
            return c[0] * np.exp(c[1] * u)

        def dN(u):
            return c[0] * c[1] * np.exp(c[1] * u)
    else:
        raise ValueError(kind)
    return N, dN


class _B:
    def __init__(self, X, terms, weight, values, fields=None):
        self.X, self.terms, self.weight, self.values, self.fields = X, terms, weight, values, fields


def newton(W, b, pde, bcs, nl, mu=1e-10, max_iter=30, tol=1e-10, c_armijo=1e-4, max_halvings=30):
    """Returns (beta, history) with history = list of dicts (resid, alpha, du_rel)."""
    N, dN = nl_funcs(*nl)
    sq = math.sqrt(mu)
    d = W.shape[1]
    zero = tuple([0] * d)
    # operator rows of L at the PDE points (for L[u_N] = A_L beta)
    AL, _, _ = assemble(W, b, [_B(pde.X, pde.terms, 1.0, None)], want_scale=False)
    # warm start: linear part only
    A0, r0, _ = assemble(W, b, [pde] + list(bcs), want_scale=False)
    beta, _, _ = lstsq_mu(A0, r0, sq)

    def state(beta):
        u = evaluate(W, b, beta, pde.X)
        Lu = AL @ beta
        neg = pde.values - Lu - N(u)
        negs = [neg]
        r2 = float(neg @ neg)
        for bc in bcs:
            nb = bc.values - evaluate(W, b, beta, bc.X)
            negs.append(nb)
            r2 += bc.weight ** 2 * float(nb @ nb)
        return u, negs, math.sqrt(r2)

    u, negs, rn = state(beta)
    hist = [{"resid": rn, "alpha": None, "du_rel": None}]
    for _ in range(max_iter):
        Jb = [_B(pde.X, list(pde.terms) + [(zero, 1.0, 0)], 1.0, negs[0], dN(u)[:, None])]
        Jb += [_B(bc.X, bc.terms, bc.weight, nb) for bc, nb in zip(bcs, negs[1:])]
        J, rhs, _ = assemble(W, b, Jb, want_scale=False)
        delta, _, _ = lstsq_mu(J, rhs, sq)
        alpha = 1.0
        for _h in range(max_halvings):
            trial = beta + alpha * delta
            u_t, negs_t, rn_t = state(trial)
            if rn_t <= (1.0 - c_armijo * alpha) * rn:
                break
            alpha *= 0.5
        du = float(np.linalg.norm(u_t - u) / max(np.linalg.norm(u_t), 1e-300))
        beta, u, negs, rn = trial, u_t, negs_t, rn_t
        hist.append({"resid": rn, "alpha": alpha, "du_rel": du})
        if du < tol:
            break
    return beta, hist
