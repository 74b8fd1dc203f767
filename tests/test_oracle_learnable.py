"""Pins of the learnable-bandwidth oracle (oracle/learnable.py; App. E), CPU only.

pin: brute force -- the analytic gradient of Lout(L) = ||A(L) beta* - b||^2 equals central
finite differences of Lout itself (each Lout evaluation = a fresh oracle assembly + Householder
solve), for the scalar bandwidth (L = sigma I) and a lower-triangular Cholesky factor."""
import numpy as np

import oracle.learnable as ol
import workloads as wl


def _setup():
    p = wl.make_helmholtz2d(n_int=300, per_edge=20, n_features=60)
    W_hat, b = p.parity_features()
    return p, W_hat, b


def test_scalar_sigma_gradient_matches_fd():
    p, W_hat, b = _setup()
    for sigma in (4.0, 6.0):          # cond(A) <~ 1e7 here, so central FD of Lout is clean
        L = sigma * np.eye(2)
        loss, G, _ = ol.outer_grad(L, W_hat, b, p.blocks)
        g = np.trace(G)                                  # dLout/dsigma with L = sigma I
        h = 1e-4 * sigma
        lp = ol.outer_loss((sigma + h) * np.eye(2), W_hat, b, p.blocks)[0]
        lm = ol.outer_loss((sigma - h) * np.eye(2), W_hat, b, p.blocks)[0]
        fd = (lp - lm) / (2 * h)
        assert abs(g - fd) <= 1e-5 * max(abs(fd), 1e-12 * loss), (sigma, g, fd)


def test_cholesky_gradient_matches_fd():
    p, W_hat, b = _setup()
    L = np.array([[3.0, 0.0], [0.7, 4.0]])
    loss, G, _ = ol.outer_grad(L, W_hat, b, p.blocks)
    for (k, l) in [(0, 0), (1, 0), (1, 1)]:
        h = 1e-5
        Lp, Lm = L.copy(), L.copy()
        Lp[k, l] += h
        Lm[k, l] -= h
        fd = (ol.outer_loss(Lp, W_hat, b, p.blocks)[0] - ol.outer_loss(Lm, W_hat, b, p.blocks)[0]) / (2 * h)
        assert abs(G[k, l] - fd) <= 1e-5 * max(abs(fd), abs(G).max()), (k, l, G[k, l], fd)


def test_gradient_with_coefficient_field_matches_fd():
    """variable-coefficient operator (k^2 (1 + x_1) u term as a coefficient field)"""
    p = wl.make_helmholtz2d_var(n_int=300, per_edge=20, n_features=60)
    W_hat, b = p.parity_features()
    L = np.array([[4.0, 0.0], [0.5, 5.0]])
    loss, G, _ = ol.outer_grad(L, W_hat, b, p.blocks)
    for (k, l) in [(0, 0), (1, 0), (1, 1)]:
        h = 1e-5
        Lp, Lm = L.copy(), L.copy()
        Lp[k, l] += h
        Lm[k, l] -= h
        fd = (ol.outer_loss(Lp, W_hat, b, p.blocks)[0] - ol.outer_loss(Lm, W_hat, b, p.blocks)[0]) / (2 * h)
        assert abs(G[k, l] - fd) <= 1e-5 * max(abs(fd), abs(G).max()), (k, l, G[k, l], fd)
    # the field matters: dropping it changes the gradient
    import dataclasses
    const = [dataclasses.replace(p.blocks[0], terms=p.blocks[0].terms[:-1] + [((0, 0), 100.0, -1)],
                                 fields=None), p.blocks[1]]
    _, G0, _ = ol.outer_grad(L, W_hat, b, const)
    assert np.abs(G0 - G).max() > 1e-3 * np.abs(G).max()


def test_ridge_augmented_gradient_matches_fd():
    """reading B2: with a Tikhonov inner solve the outer loss is ||A beta* - b||^2 + mu ||beta*||^2
    and the envelope gradient is its exact derivative -- brute force by central FD; the plain
    residual loss (without mu ||beta||^2) would NOT match at this mu"""
    p, W_hat, b = _setup()
    sq = 3e-2
    L = np.array([[3.0, 0.0], [0.7, 4.0]])
    loss, G, beta = ol.outer_grad(L, W_hat, b, p.blocks, sqrt_mu=sq)
    for (k, l) in [(0, 0), (1, 0), (1, 1)]:
        h = 1e-5
        Lp, Lm = L.copy(), L.copy()
        Lp[k, l] += h
        Lm[k, l] -= h
        fd = (ol.outer_loss(Lp, W_hat, b, p.blocks, sqrt_mu=sq)[0]
              - ol.outer_loss(Lm, W_hat, b, p.blocks, sqrt_mu=sq)[0]) / (2 * h)
        assert abs(G[k, l] - fd) <= 1e-5 * max(abs(fd), abs(G).max()), (k, l, G[k, l], fd)
    # the residual part alone differs from its FD by the dropped -2 mu beta^T dbeta/dL term
    def res_only(Lm_):
        lo, _, bt, _ = ol.outer_loss(Lm_, W_hat, b, p.blocks, sqrt_mu=sq)
        return lo - sq * sq * float(bt @ bt)
    h = 1e-5
    Lp, Lm = L.copy(), L.copy()
    Lp[1, 1] += h
    Lm[1, 1] -= h
    fd_res = (res_only(Lp) - res_only(Lm)) / (2 * h)
    assert abs(G[1, 1] - fd_res) > 1e-3 * abs(G).max()
