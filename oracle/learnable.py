"""Oracle for learnable-bandwidth Fast-LSQ (App. E) -- TEST INFRASTRUCTURE ONLY.

Outer loss Lout(L) = ||A(L) beta* - b||^2 with W = L W^, A by the oracle's
term-by-term assembly, beta* by its Householder lstsq.  The gradient is written out from the
definition: for each term c(x) prod W^e Phi_p(W.x + b) (e, p from the symbolic differentiator;
c(x) = coef, or coef times a coefficient field),
    d/dW_k = c e_k prod W^(e - e_k) Phi_p(z) + c prod W^e x_k Phi_{p+1}(z),
    dLout/dL_kl = 2 sum_ij r_i beta_j dA_ij/dW_jk W^_jl      (beta* optimal: envelope)
evaluated with numpy sin / cos on the full (rows x features) grid -- small inputs only.
With a Tikhonov inner solve (sqrt_mu > 0) the outer loss is the ridge-augmented
    Lout_mu = ||A beta* - b||^2 + mu ||beta*||^2    (reading B2)
-- the objective beta* minimises -- so the same envelope formula is its exact gradient (mu
||beta||^2 has no explicit L dependence); at mu = 0 it is Lout.
Pinned by central finite differences of Lout / Lout_mu (tests/test_oracle_learnable.py).
"""
from __future__ import annotations

import math

import numpy as np

from . import assemble, diff, lstsq, lstsq_mu


def _phi(p, z):
    return [np.sin, np.cos, lambda t: -np.sin(t), lambda t: -np.cos(t)][p % 4](z)


def outer_loss(Lmat, W_hat, b, blocks, sqrt_mu=0.0, normalize=True):
    W = W_hat @ np.asarray(Lmat, float).T            # W_j = L W^_j
    A, rhs, _ = assemble(W, b, blocks, want_scale=False, normalize=normalize)
    if sqrt_mu > 0:
        beta, _, _ = lstsq_mu(A, rhs, sqrt_mu)
    else:
        beta, _, _ = lstsq(A, rhs)
    r = A @ beta - rhs
    loss = float(r @ r)
    if sqrt_mu > 0:                                  # reading B2: the inner solve's objective
        loss += sqrt_mu * sqrt_mu * float(beta @ beta)
    return loss, W, beta, r


def outer_grad(Lmat, W_hat, b, blocks, sqrt_mu=0.0, normalize=True):
    loss, W, beta, r = outer_loss(Lmat, W_hat, b, blocks, sqrt_mu, normalize)
    F, d = W.shape
    s = 1.0 / math.sqrt(F) if normalize else 1.0
    V = np.zeros((F, d))                             # V_jk = sum_i r_i dA_ij / dW_jk
    off = 0
    for blk in blocks:
        X = np.asarray(blk.X, float)
        n = X.shape[0]
        ri = r[off:off + n]
        off += n
        Z = X @ W.T + b                              # (n, F)
        fields = getattr(blk, "fields", None)
        for alpha, coef, field in blk.terms:
            # per-row coefficient c_t(x_i): coef, times the coefficient field for field terms
            rc = ri * (fields[:, field] if field >= 0 else 1.0)
            e, p = diff(alpha)
            mono = np.ones(F)
            for k in range(d):
                mono = mono * W[:, k] ** e[k]
            phase_p = _phi(p, Z)
            phase_p1 = _phi(p + 1, Z)
            for k in range(d):
                # c e_k prod W^(e - e_k) Phi_p(z)
                if e[k] > 0:
                    m_k = np.ones(F)
                    for l in range(d):
                        m_k = m_k * W[:, l] ** (e[l] - (1 if l == k else 0))
                    V[:, k] += blk.weight * s * coef * e[k] * m_k * (rc @ phase_p)
                # c prod W^e x_k Phi_{p+1}(z)
                V[:, k] += blk.weight * s * coef * mono * ((rc * X[:, k]) @ phase_p1)
    G = 2.0 * np.einsum("jk,j,jl->kl", V, beta, W_hat)
    return loss, G, beta
