"""Oracle Newton-Raphson for L[u] + N(u, Du) = f (Eq. 4-5) -- TEST INFRASTRUCTURE ONLY.

Step by step in the paper's order (readings N1-N5 in DESIGN.md §3):
  warm start  : beta_0 = Tikhonov lstsq of the linear part (N dropped)
  residual    : R = [(L + N)[u_N](x_i) - f_i ; lam (u_N(x_b) - g_b)]
  Jacobian    : J = [L[phi_j](x_i) + N_u(x_i) s phi_j(x_i) + N_Du(x_i) D phi_j(x_i) ;
                     lam s phi_j(x_b)]
  step        : delta = argmin ||J delta + R||^2 + mu ||delta||^2, mu = 1e-10
  line search : alpha = 1, halve while ||R(beta + alpha delta)|| > (1 - c alpha)||R(beta)||,
                c = 1e-4 (Armijo sufficient decrease on the residual norm)
  stop        : ||u_{k+1} - u_k|| / ||u_{k+1}|| < tol at the collocation points
  continuation: a parameter schedule, each stage warm-started from the previous
Nonlinearities: ('poly', coefs), ('exp', [a0, a1]), ('udu', [a0], alpha) = a0 u D^alpha u.
Primitives: orc_assemble (term-by-term closed form), orc_lstsq_mu (Householder QR),
orc_eval, numpy matrix-vector products and the pointwise N and its partial derivatives.
"""
from __future__ import annotations

import math

import numpy as np

from . import assemble, evaluate, lstsq_mu


def nl_funcs(kind, coefs):
    """pointwise kinds: (N(u), dN/du(u))"""
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


def newton(W, b, pde, bcs, nl, mu=1e-10, max_iter=30, tol=1e-10, c_armijo=1e-4, max_halvings=30,
           beta0=None):
    """Returns (beta, history) with history = list of dicts (resid, alpha, du_rel)."""
    kind, coefs = nl[0], nl[1]
    quasi = kind == "udu"
    alpha_d = tuple(nl[2]) if quasi else None
    sq = math.sqrt(mu)
    d = W.shape[1]
    zero = tuple([0] * d)
    # operator rows at the PDE points: L[u_N] = A_L beta, D^alpha u_N = A_D beta
    AL, _, _ = assemble(W, b, [_B(pde.X, pde.terms, 1.0, None)], want_scale=False)
    AD = assemble(W, b, [_B(pde.X, [(alpha_d, 1.0, -1)], 1.0, None)], want_scale=False)[0] if quasi else None
    if beta0 is None:
        A0, r0, _ = assemble(W, b, [pde] + list(bcs), want_scale=False)
        beta, _, _ = lstsq_mu(A0, r0, sq)
    else:
        beta = np.array(beta0, dtype=float)

    def state(beta):
        u = evaluate(W, b, beta, pde.X)
        Lu = AL @ beta
        if quasi:
            Du = AD @ beta
            N = coefs[0] * u * Du
            fields = np.stack([coefs[0] * Du, coefs[0] * u], axis=1)     # dN/du, dN/dDu
        else:
            Nf, dNf = nl_funcs(kind, coefs)
            N = Nf(u)
            fields = dNf(u)[:, None]
        neg = pde.values - Lu - N
        negs = [neg]
        r2 = float(neg @ neg)
        for bc in bcs:
            nb = bc.values - evaluate(W, b, beta, bc.X)
            negs.append(nb)
            r2 += bc.weight ** 2 * float(nb @ nb)
        return u, fields, negs, math.sqrt(r2)

    u, fields, negs, rn = state(beta)
    hist = [{"resid": rn, "alpha": None, "du_rel": None}]
    for _ in range(max_iter):
        terms = list(pde.terms) + [(zero, 1.0, 0)]
        if quasi:
            terms.append((alpha_d, 1.0, 1))
        Jb = [_B(pde.X, terms, 1.0, negs[0], fields)]
        Jb += [_B(bc.X, bc.terms, bc.weight, nb) for bc, nb in zip(bcs, negs[1:])]
        J, rhs, _ = assemble(W, b, Jb, want_scale=False)
        delta, _, _ = lstsq_mu(J, rhs, sq)
        alpha = 1.0
        for _h in range(max_halvings):
            trial = beta + alpha * delta
            u_t, fields_t, negs_t, rn_t = state(trial)
            if rn_t <= (1.0 - c_armijo * alpha) * rn:
                break
            alpha *= 0.5
        du = float(np.linalg.norm(u_t - u) / max(np.linalg.norm(u_t), 1e-300))
        beta, u, fields, negs, rn = trial, u_t, fields_t, negs_t, rn_t
        hist.append({"resid": rn, "alpha": alpha, "du_rel": du})
        if du < tol:
            break
    return beta, hist


def continuation(W, b, make_pde, bcs, nl, schedule, **kw):
    beta, hists = None, []
    for p in schedule:
        beta, h = newton(W, b, make_pde(p), bcs, nl, beta0=beta, **kw)
        hists.append(h)
    return beta, hists
