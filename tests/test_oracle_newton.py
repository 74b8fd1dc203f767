"""Pins of the oracle Newton-Raphson (oracle/newton.py) -- CPU only.

pins: manufactured nonlinear solutions recovered (closed-form u*); with N = 0 the method is
the linear Fast-LSQ solve (warm start already optimal: the first Newton step changes u by
~nothing); the pointwise N' agrees with central differences of N; the residual norm decreases
monotonically under the Armijo rule; the early iterations contract quadratically.
"""
import numpy as np
import pytest

import oracle
import oracle.newton as on
import workloads as wl


@pytest.mark.parametrize("name", wl.NL_NAMES)
def test_newton_recovers_manufactured_solution(name):
    p = wl.make_nl_problem(name)
    W, b = p.parity_features()
    beta, hist = on.newton(W, b, p.blocks[0], p.blocks[1:], p.nl, max_iter=10, tol=1e-8)
    Xt = p.test_points(2000)
    u = oracle.evaluate(W, b, beta, Xt)
    us = p.u_star(Xt)
    assert np.linalg.norm(u - us) / np.linalg.norm(us) < 1e-6
    res = [h["resid"] for h in hist]
    assert all(r1 <= r0 * (1 + 1e-12) for r0, r1 in zip(res, res[1:]))
    du = [h["du_rel"] for h in hist[1:]]
    assert du[1] < 0.1 * du[0] and du[2] < 0.1 * du[1]        # fast (quadratic-phase) contraction


def test_newton_with_zero_nonlinearity_is_linear_solve():
    p = wl.make_nl_problem("nl_poisson2d")
    W, b = p.parity_features()
    # same rows, N = 0: f must then be -Lap u* only
    pde = p.blocks[0]
    x, y = pde.X[:, 0], pde.X[:, 1]
    pde.values = 2 * np.pi ** 2 * np.sin(np.pi * x) * np.sin(np.pi * y)
    beta, hist = on.newton(W, b, pde, p.blocks[1:], ("poly", [0.0]), max_iter=3, tol=0.0)
    assert hist[1]["du_rel"] < 1e-7          # only the Tikhonov bias moves (mu = 1e-10)
    A, r, _ = oracle.assemble(W, b, [pde] + p.blocks[1:], want_scale=False)
    b0, _, _ = oracle.lstsq_mu(A, r, 1e-5)
    Xt = p.test_points(500)
    u0 = oracle.evaluate(W, b, b0, Xt)
    u1 = oracle.evaluate(W, b, beta, Xt)
    assert np.linalg.norm(u1 - u0) / np.linalg.norm(u0) < 1e-8


def test_nonlinearity_derivatives_fd():
    u = np.linspace(-2, 2, 41)
    h = 1e-6
    for spec in [("poly", [0.3, -1.0, 0.5, 1.0]), ("exp", [-1.0, 1.0]), ("exp", [2.0, -0.5])]:
        N, dN = on.nl_funcs(*spec)
        fd = (N(u + h) - N(u - h)) / (2 * h)
        assert np.allclose(dN(u), fd, rtol=1e-7, atol=1e-7)


def test_lstsq_mu_matches_stacked_library():
    g = np.random.default_rng(3)
    A = g.normal(size=(40, 12))
    bv = g.normal(size=40)
    sq = 0.3
    beta, _, _ = oracle.lstsq_mu(A, bv, sq)
    ref, *_ = np.linalg.lstsq(np.vstack([A, sq * np.eye(12)]), np.concatenate([bv, np.zeros(12)]),
                              rcond=None)
    assert np.allclose(beta, ref, rtol=1e-10, atol=1e-12)


def test_burgers_continuation_recovers_exact_solution():
    """pin: closed form -- steady viscous Burgers -nu u'' + u u' = 0 has u* = -tanh(x/(2 nu));
    continuation nu = 1 -> 0.5 -> 0.2 with the quasi-linear u u_x Jacobian."""
    p, mk = wl.make_burgers1d()
    W, b = p.parity_features()
    beta, hs = on.continuation(W, b, mk, p.blocks[1:], p.nl, [1.0, 0.5, 0.2], max_iter=8, tol=1e-9)
    Xt = p.test_points(1000)
    u = oracle.evaluate(W, b, beta, Xt)
    us = p.u_star(Xt)
    assert np.linalg.norm(u - us) / np.linalg.norm(us) < 1e-5
    assert len(hs) == 3 and hs[-1][-1]["resid"] < hs[-1][0]["resid"]
