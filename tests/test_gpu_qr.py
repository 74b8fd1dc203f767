"""libfls's blocked Householder QR (fls_geqrf; the factorisation behind fls_solve, fls_qr_factor,
fls_qr_r) against the mathematics: Q R = A and Q^T Q = I to rounding, |diag R| equal to
cuSOLVER geqrf's (torch.geqrf) on full-rank inputs, tau = 0 for an already-zero column, and the
LAPACK storage format (torch.linalg.householder_product rebuilds Q from it)."""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2602_10541_b200 import fls


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return fls.Context()


@pytest.fixture(params=["blocked", "cusolver"], autouse=True)
def method(request, monkeypatch):
    """every test runs on libfls's blocked QR and on the cuSOLVER path (same storage format)"""
    monkeypatch.setenv("FLS_QR", request.param)
    return request.param


def _factor(ctx, A, pad=3):
    m, n = A.shape
    lda = m + pad
    M = torch.zeros((n, lda), dtype=torch.float64, device="cuda")
    M[:, :m] = A.T
    tau = fls.fls_geqrf(ctx, M.view(-1), m, lda, n)
    torch.cuda.synchronize()
    assert torch.all(M[:, m:] == 0), "rows past n_rows (lda padding) were written"
    return M[:, :m].T.contiguous(), tau


def _check(A, a, tau, tol=1e-13):
    m, n = A.shape
    k = min(m, n)
    Q = torch.linalg.householder_product(a[:, :k], tau)          # m x k
    R = torch.triu(a[:k, :])
    nA = torch.linalg.norm(A)
    assert float(torch.linalg.norm(Q @ R - A) / nA) <= tol
    assert float(torch.linalg.norm(Q.T @ Q - torch.eye(k, dtype=A.dtype, device=A.device))) <= tol * k ** 0.5


@pytest.mark.parametrize("m,n", [(100, 37), (1000, 300), (3000, 700), (777, 513), (20000, 1100),
                                 (64, 64), (33, 1), (1, 5), (300, 520), (40, 100),
                                 (300000, 100)])   # tall: leaves narrower than 32 (slab budget)
def test_geqrf_reconstructs_and_matches_cusolver_diag(ctx, m, n):
    g = torch.Generator(device="cuda").manual_seed(m * 1000 + n)
    A = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g)
    a, tau = _factor(ctx, A)
    _check(A, a, tau)
    a_ref, _ = torch.geqrf(A)
    k = min(m, n)
    d, d_ref = a.diagonal()[:k].abs(), a_ref.diagonal()[:k].abs()
    assert float(((d - d_ref).abs() / d_ref).max()) <= 1e-10


def test_geqrf_rank_deficient_and_zero_columns(ctx):
    g = torch.Generator(device="cuda").manual_seed(7)
    m, n = 2500, 600
    B = torch.randn((m, 150), dtype=torch.float64, device="cuda", generator=g)
    A = B @ torch.randn((150, n), dtype=torch.float64, device="cuda", generator=g)  # rank 150
    A[:, 5] = 0.0                      # zero column: tau_5 = 0, H_5 = I
    A[:, 300] = A[:, 299]              # duplicate column
    a, tau = _factor(ctx, A)
    _check(A, a, tau, tol=1e-12)
    assert float(tau[5]) == 0.0
    d = a.diagonal().abs()
    nA = float(torch.linalg.norm(A))
    assert float(d[160:].max()) <= 1e-11 * nA          # numerical rank shows on the diagonal


def test_geqrf_solves_least_squares_like_lstsq(ctx):
    """[A | b] factored together: R beta = (Q^T b)[0:n] is the LAPACK least-squares solution and
    |R(n, n)| the residual norm (how fls_solve uses it)"""
    g = torch.Generator(device="cuda").manual_seed(11)
    m, n = 5000, 800
    A = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn((m, 1), dtype=torch.float64, device="cuda", generator=g)
    a, _ = _factor(ctx, torch.cat([A, b], 1))
    beta = torch.linalg.solve_triangular(torch.triu(a[:n, :n]), a[:n, n:], upper=True)
    ref = torch.linalg.lstsq(A.cpu(), b.cpu()).solution.cuda()
    assert float(torch.linalg.norm(beta - ref) / torch.linalg.norm(ref)) <= 1e-11
    res = float(torch.linalg.norm(A @ ref - b))
    assert abs(abs(float(a[n, n])) - res) <= 1e-10 * res


def test_geqrf_errors(ctx):
    M = torch.zeros(100, dtype=torch.float64, device="cuda")
    with pytest.raises(fls.FlsError):
        fls.fls_geqrf(ctx, M, 10, 5, 3)                 # lda < n_rows
    with pytest.raises(fls.FlsError):
        fls.fls_geqrf(ctx, M, 0, 10, 3)


@pytest.mark.parametrize("name,size", [("c1_poisson1d", "full"), ("c2_poisson2d", "full"),
                                       ("c5_biharm3d", "mini")])
def test_solve_parity_with_oracle_on_both_qr_paths(ctx, name, size):
    """fls_solve (assembly -> QR -> trsv) on numerically rank-deficient systems (C1: rank ~41 of
    500) and with the relative ridge (C5): fitted u vs the oracle chain <= 1e-6 on either path"""
    import math

    import numpy as np

    import oracle
    import workloads as wl
    from gpu_common import U_TOL, dev_blocks
    p = wl.make_problem(name, size)
    W, b = p.parity_features()
    Wd, bd = torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda()
    F, R = p.n_features, p.n_rows
    ridge = p.ridge_rel > 0
    Ab, lda = fls.fls_assemble(ctx, Wd, bd, dev_blocks(p), extra_rows=F if ridge else 0)
    beta, _ = fls.fls_solve(ctx, Ab, R, lda, F, p.ridge_rel)
    Xt = p.test_points(10_000)
    u_gpu = fls.fls_eval(ctx, Wd, bd, beta, torch.from_numpy(Xt).cuda()).cpu().numpy()
    Ao, ro, _ = oracle.assemble(W, b, p.blocks, want_scale=False)
    beta_o, _, _ = oracle.lstsq(Ao, ro, ridge_rel=p.ridge_rel)
    u_orc = oracle.evaluate(W, b, beta_o, Xt)
    assert np.linalg.norm(u_gpu - u_orc) / np.linalg.norm(u_orc) <= U_TOL


@pytest.mark.parametrize("P,kb,n,ridge", [(4, 301, 300, 0.0), (8, 301, 300, 1e-3), (3, 150, 300, 1e-2),
                                          (2, 1101, 1100, 0.0), (5, 1101, 1100, 1e-4),
                                          (1, 1101, 1100, 0.0), (1, 1101, 1100, 1e-3)])
def test_solve_stacked_matches_dense_solve(ctx, P, kb, n, ridge):
    """fls_solve_stacked (row-permuted stack, panels stopped where the triangles end) == fls_solve
    on the same stack in block order: beta and |R(F, F)| (full column rank inputs)"""
    F = n - 1
    g = torch.Generator(device="cuda").manual_seed(P * 1000 + kb)
    lds = P * kb
    S = torch.zeros(((F + 1) * lds,), dtype=torch.float64, device="cuda")
    Sv = S.view(F + 1, lds)
    for r in range(P):
        k = min(kb, F + 1)
        B = torch.randn((k, F + 1), dtype=torch.float64, device="cuda", generator=g)
        B.diagonal().add_(4.0 * math.sqrt(F))      # well conditioned: random triangles are not
        Sv[:, r * kb:r * kb + k] = torch.triu(B).T        # upper-trapezoidal factor of block r
    fro = float(torch.linalg.norm(Sv[:F, :]))
    sq = ridge * fro
    beta_s, res_s = fls.fls_solve_stacked(ctx, S, P, kb, lds, F, sq)
    ld = ((lds + F + 3) // 4) * 4
    M = torch.zeros(((F + 1) * ld,), dtype=torch.float64, device="cuda")
    M.view(F + 1, ld)[:, :lds] = Sv
    beta_d, res_d = fls.fls_solve_mu(ctx, M, lds, ld, F, sq)
    assert float(torch.linalg.norm(beta_s - beta_d) / torch.linalg.norm(beta_d)) <= 1e-10
    assert abs(res_s - res_d) <= 1e-10 * max(res_d, 1e-300)
    assert torch.equal(Sv[:, :1], S.view(F + 1, lds)[:, :1])   # S not modified (spot check)


@pytest.mark.parametrize("m,n,ridge", [(3000, 700, 1e-3), (5000, 1100, 1e-4), (2500, 1100, 0.0)])
def test_cached_qr_with_ridge_matches_stacked_lstsq(ctx, m, n, ridge):
    """fls_qr_factor + fls_qr_solve (ormqr on the stored reflectors, grouped mode for the ridge
    rows on the blocked path) == LAPACK lstsq of [A; sqrt_mu I] for several right-hand sides"""
    g = torch.Generator(device="cuda").manual_seed(m + n)
    A = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn((m, 3), dtype=torch.float64, device="cuda", generator=g)
    sq = ridge * float(torch.linalg.norm(A))
    qr = fls.QRFactor(ctx, A.T.contiguous().view(-1), m, m, n, sq)
    Beta = qr.solve(B.T.contiguous().view(-1), m)                      # (3, n)
    qr.close()
    As = torch.cat([A, sq * torch.eye(n, dtype=torch.float64, device="cuda")]).cpu()
    Bs = torch.cat([B, torch.zeros((n, 3), dtype=torch.float64, device="cuda")]).cpu()
    ref = torch.linalg.lstsq(As, Bs).solution.T.cuda()
    assert float(torch.linalg.norm(Beta - ref) / torch.linalg.norm(ref)) <= 1e-9


def test_solve_zero_column_is_erank(ctx):
    """an exactly zero column gives an exactly zero diagonal of R: fls_solve reports FLS_ERANK
    (mu = 0) on either QR path, and solves with a ridge"""
    m, n = 2000, 1100
    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g)
    A[:, 17] = 0.0
    ld = ((m + n + 3) // 4) * 4
    M = torch.zeros(((n + 1) * ld,), dtype=torch.float64, device="cuda")
    M.view(n + 1, ld)[:n, :m] = A.T
    M.view(n + 1, ld)[n, :m] = torch.randn(m, dtype=torch.float64, device="cuda", generator=g)
    M2 = M.clone()
    with pytest.raises(fls.FlsError, match="ERANK"):
        fls.fls_solve(ctx, M, m, ld, n, 0.0)
    beta, _ = fls.fls_solve_mu(ctx, M2, m, ld, n, 1e-6)
    assert bool(torch.isfinite(beta).all()) and abs(float(beta[17])) <= 1e-6 * float(beta.abs().max())
