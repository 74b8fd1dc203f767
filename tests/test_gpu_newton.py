"""GPU Newton-Raphson (paper_2602_10541_b200.newton over libfls) vs the oracle Newton
(oracle/newton.py), same algorithm and parameters: fitted u at held-out points within 1e-6,
pointwise residual / N' kernel against numpy."""
import numpy as np
import pytest
import torch

import oracle
import oracle.newton as on
import workloads as wl
from gpu_common import U_TOL, dev_blocks

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2602_10541_b200 import fls
    from paper_2602_10541_b200.newton import solve_nonlinear


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return fls.Context()


@pytest.mark.parametrize("spec", [("poly", [0.3, -1.0, 0.5, 1.0]), ("exp", [-1.0, 1.0])])
def test_nl_residual_kernel(ctx, spec):
    g = np.random.default_rng(1)
    n = 10_007
    u, Lu, f, up = (g.normal(size=n) for _ in range(4))
    N, dN = on.nl_funcs(*spec)
    T = [torch.from_numpy(v).cuda() for v in (u, Lu, f, up)]
    neg, dn, st = fls.fls_nl_residual(ctx, fls.make_nonlinearity(*spec), T[1], T[0], T[2], u_prev=T[3])
    ref = f - Lu - N(u)
    assert np.allclose(neg.cpu().numpy(), ref, rtol=1e-13, atol=1e-13 * np.abs(ref).max())
    assert np.allclose(dn.cpu().numpy(), dN(u), rtol=1e-13, atol=1e-13)
    assert abs(st[0] - (ref @ ref)) <= 1e-11 * (ref @ ref)
    assert abs(st[1] - (u @ u)) <= 1e-12 * (u @ u)
    assert abs(st[2] - ((u - up) @ (u - up))) <= 1e-12 * ((u - up) @ (u - up))
    out = fls.fls_axpy(ctx, 0.37, T[0], T[1]).cpu().numpy()
    assert np.allclose(out, Lu + 0.37 * u, rtol=1e-15, atol=1e-15)


@pytest.mark.parametrize("name", wl.NL_NAMES)
def test_newton_parity_with_oracle(ctx, name):
    p = wl.make_nl_problem(name)
    W, b = p.parity_features()
    Wd, bd = torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda()
    blocks = dev_blocks(p)
    beta, hist = solve_nonlinear(ctx, Wd, bd, blocks[0], blocks[1:], *p.nl, max_iter=10, tol=1e-8)
    beta_o, hist_o = on.newton(W, b, p.blocks[0], p.blocks[1:], p.nl, max_iter=10, tol=1e-8)
    Xt = p.test_points(2000)
    u_gpu = fls.fls_eval(ctx, Wd, bd, beta, torch.from_numpy(Xt).cuda()).cpu().numpy()
    u_orc = oracle.evaluate(W, b, beta_o, Xt)
    assert np.linalg.norm(u_gpu - u_orc) / np.linalg.norm(u_orc) <= U_TOL
    assert abs(len(hist) - len(hist_o)) <= 1
    for h, ho in zip(hist[:3], hist_o[:3]):                 # same residual trajectory early on
        assert abs(h["resid"] - ho["resid"]) <= 1e-6 * ho["resid"] + 1e-9
    us = p.u_star(Xt)
    assert np.linalg.norm(u_gpu - us) / np.linalg.norm(us) < 1e-6


def test_burgers_continuation_parity(ctx):
    """quasi-linear N = u u_x (FLS_NL_UDU) + continuation nu = 1 -> 0.5 -> 0.2:
    GPU vs oracle after the same schedule, and both vs u* = -tanh(x / 0.4)"""
    from paper_2602_10541_b200.newton import solve_continuation
    p, mk = wl.make_burgers1d()
    W, b = p.parity_features()
    Wd, bd = torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda()
    bcs = dev_blocks(p)[1:]

    def mk_dev(nu):
        blk = mk(nu)
        return fls.Block(torch.from_numpy(blk.X).cuda(), blk.terms, blk.weight,
                         torch.from_numpy(blk.values).cuda())
    beta, hs = solve_continuation(ctx, Wd, bd, mk_dev, bcs, "udu", [1.0], [1.0, 0.5, 0.2],
                                  nl_alpha=(1,), max_iter=8, tol=1e-9)
    beta_o, hs_o = on.continuation(W, b, mk, p.blocks[1:], p.nl, [1.0, 0.5, 0.2], max_iter=8,
                                   tol=1e-9)
    Xt = p.test_points(1000)
    u_gpu = fls.fls_eval(ctx, Wd, bd, beta, torch.from_numpy(Xt).cuda()).cpu().numpy()
    u_orc = oracle.evaluate(W, b, beta_o, Xt)
    assert np.linalg.norm(u_gpu - u_orc) / np.linalg.norm(u_orc) <= U_TOL
    us = p.u_star(Xt)
    assert np.linalg.norm(u_gpu - us) / np.linalg.norm(us) < 1e-5
    assert [len(h) for h in hs] == [len(h) for h in hs_o] or all(abs(len(a) - len(c)) <= 1 for a, c in zip(hs, hs_o))


def test_udu_residual_kernel(ctx):
    g = np.random.default_rng(3)
    n = 5003
    u, Lu, Du, f = (g.normal(size=n) for _ in range(4))
    T = [torch.from_numpy(v).cuda() for v in (u, Lu, Du, f)]
    neg, dNu, dNd, st = fls.fls_nl_residual2(ctx, fls.make_nonlinearity("udu", [0.7]), T[1], T[0],
                                             T[2], T[3])
    ref = f - Lu - 0.7 * u * Du
    assert np.allclose(neg.cpu().numpy(), ref, rtol=1e-14, atol=1e-14)
    assert np.allclose(dNu.cpu().numpy(), 0.7 * Du, rtol=1e-15, atol=0)
    assert np.allclose(dNd.cpu().numpy(), 0.7 * u, rtol=1e-15, atol=0)


def test_newton_uses_the_bc_operator_in_residual_and_jacobian(ctx):
    """a Robin boundary operator (u + 0.3 du/dx on the x-edges): with N = 0 the linear warm start
    is already the Tikhonov least-squares solution, so Newton must stop there -- its residual is
    evaluated with the same BC operator the Jacobian rows use (a residual taken with the identity
    would move beta away).  Compared with one direct solve of the stacked system."""
    import math
    g = np.random.default_rng(3)
    n, nb, F = 900, 120, 250
    Xi_h = g.random((n, 2))
    Xb_h = np.stack([np.repeat([0.0, 1.0], nb // 2), g.random(nb)], 1)
    # manufactured u* = sin(x + 0.5) cos(y): -Lap u* = 2 u*, Robin data u* + 0.3 du*/dx
    us = lambda X: np.sin(X[:, 0] + 0.5) * np.cos(X[:, 1])
    usx = lambda X: np.cos(X[:, 0] + 0.5) * np.cos(X[:, 1])
    Xi, Xb = torch.from_numpy(Xi_h).cuda(), torch.from_numpy(Xb_h).cuda()
    f = torch.from_numpy(2.0 * us(Xi_h)).cuda()
    gb = torch.from_numpy(us(Xb_h) + 0.3 * usx(Xb_h)).cuda()
    lap = [((2, 0), -1.0, -1), ((0, 2), -1.0, -1)]
    robin = [((0, 0), 1.0, -1), ((1, 0), 0.3, -1)]
    # Dirichlet (identity) rows on the y-edges complete the boundary
    Xd_h = np.stack([g.random(nb), np.repeat([0.0, 1.0], nb // 2)], 1)
    Xd = torch.from_numpy(Xd_h).cuda()
    pde = fls.Block(Xi, lap, 1.0, f)
    bc = fls.Block(Xb, robin, 10.0, gb)
    bcd = fls.Block(Xd, [((0, 0), 1.0, -1)], 10.0, torch.from_numpy(us(Xd_h)).cuda())
    W, b = fls.fls_features(ctx, 2, F, 3.0, 0)
    beta, hist = solve_nonlinear(ctx, W, b, pde, [bc, bcd], "poly", [0.0], mu=1e-10, max_iter=3)
    R = n + 2 * nb
    lda = fls.round_up(R + F, 4)
    Ab = torch.empty(((F + 1) * lda,), dtype=torch.float64, device="cuda")
    fls.fls_assemble(ctx, W, b, [pde, bc, bcd], A=Ab, lda=lda)
    beta_d, res_d = fls.fls_solve_mu(ctx, Ab, R, lda, F, math.sqrt(1e-10))
    Xt_h = g.random((2000, 2))
    Xt = torch.from_numpy(Xt_h).cuda()
    u = fls.fls_eval(ctx, W, b, beta, Xt).cpu().numpy()
    u_d = fls.fls_eval(ctx, W, b, beta_d, Xt).cpu().numpy()
    assert np.linalg.norm(u_d - us(Xt_h)) <= 1e-5 * np.linalg.norm(us(Xt_h))   # well posed
    assert np.linalg.norm(u - u_d) <= 1e-6 * np.linalg.norm(u_d)    # an identity-BC residual moves it O(1)
    # the residual Newton reports at its warm start (= beta_d) is ||A beta - b|| of the stacked
    # system WITH the Robin rows -- A beta from fls_eval_block, i.e. the assembled operators
    r2 = 0.0
    for blk in (pde, bc, bcd):
        Ab_ = fls.fls_eval_block(ctx, W, b, beta_d, blk).cpu().numpy()
        r2 += float(np.sum((Ab_ - blk.weight * blk.values.cpu().numpy()) ** 2))
    assert abs(hist[0]["resid"] - math.sqrt(r2)) <= 1e-6 * math.sqrt(r2)
