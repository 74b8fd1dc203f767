"""Pins of the CPU oracle to facts other than itself (CPU only, -m "not gpu").

Each test names what fixes the expected value: a closed form of the paper, a worked value
(tests/golden/), a library routine (numpy / scipy), brute force (finite differences), an
invariant, or a statistical law.  DESIGN.md §5 maps every oracle function to its pins.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
from scipy import stats

import oracle
import workloads as wl

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


class Blk:
    """minimal block record for oracle.assemble"""

    def __init__(self, X, terms, weight=1.0, values=None, fields=None):
        self.X = np.ascontiguousarray(X, float)
        self.terms = terms
        self.weight = weight
        self.values = values if values is not None else np.zeros(self.X.shape[0])
        self.fields = fields


def col(W, b, X, terms, normalize=False, fields=None, weight=1.0):
    A, _, S = oracle.assemble(W, b, [Blk(X, terms, weight, fields=fields)], normalize=normalize)
    return A, S


def rand_basis(d, F, sigma, seed):
    g = np.random.default_rng(seed)
    return g.normal(0, sigma, (F, d)), g.uniform(0, 2 * np.pi, F)


# ----------------------------------------------------------------------------- RNG / features
def test_philox_matches_numpy_library():
    """pin: numpy.random.Philox (Philox4x64-10) is the library routine of the same generator"""
    for seed, stream in [(0, 1), (0, 2), (5, 7), (2**63 + 11, 3)]:
        ref = np.random.Philox(key=seed + (stream << 64)).random_raw(103)
        got = oracle.raw_stream(seed, stream, 0, 103)
        assert np.array_equal(ref.astype(np.uint64), got)
    # an offset start equals the tail of the stream
    ref = np.random.Philox(key=9 + (1 << 64)).random_raw(50)
    assert np.array_equal(ref[17:], oracle.raw_stream(9, 1, 17, 33))


def test_features_deterministic_and_distribution():
    """pins: same seed -> identical bytes; W ~ N(0, sigma^2) (KS test, moments),
    b ~ U[0, 2pi) (KS test) -- P:L82."""
    d, F, sigma = 3, 40000, 3.0
    W1, b1 = oracle.features(d, F, sigma, seed=0)
    W2, b2 = oracle.features(d, F, sigma, seed=0)
    assert W1.tobytes() == W2.tobytes() and b1.tobytes() == b2.tobytes()
    W3, _ = oracle.features(d, F, sigma, seed=1)
    assert not np.array_equal(W1, W3)
    w = W1.ravel()
    n = w.size
    assert abs(w.mean()) < 5 * sigma / math.sqrt(n)
    assert abs(w.var() - sigma**2) < 5 * sigma**2 * math.sqrt(2.0 / n)
    assert stats.kstest(w / sigma, "norm").pvalue > 1e-4
    assert b1.min() >= 0.0 and b1.max() < 2 * np.pi
    assert stats.kstest(b1 / (2 * np.pi), "uniform").pvalue > 1e-4
    # odd normal count (F*d odd): last normal from the cos branch only
    W5, _ = oracle.features(1, 7, 1.0, seed=0)
    W6, _ = oracle.features(1, 8, 1.0, seed=0)
    assert np.array_equal(W5[:, 0], W6[:7, 0])


def test_features_blocks_pins():
    """pins: one block == orc_features (same streams); per-block W ~ N(0, sigma_q^2)
    (KS test per block, P:L85 multi-block bandwidths); b identical to the one-block draw."""
    W1, b1 = oracle.features(2, 3000, 1.7, seed=4)
    Wb, bb = oracle.features_blocks(2, [3000], [1.7], seed=4)
    assert np.array_equal(W1, Wb) and np.array_equal(b1, bb)
    counts, sig = [20000, 5, 30000], [0.5, 3.0, 8.0]
    W, b = oracle.features_blocks(3, counts, sig, seed=9)
    Wu, bu = oracle.features(3, sum(counts), 1.0, seed=9)
    assert np.array_equal(b, bu)
    off = 0
    for n, s in zip(counts, sig):
        blk = W[off:off + n]
        assert np.array_equal(blk, s * Wu[off:off + n])      # same normals, scaled by sigma_q
        if n > 100:
            assert stats.kstest(blk.ravel() / s, "norm").pvalue > 1e-4
        off += n


def test_kernel_limit_has_factor_half():
    """pin: random-Fourier-feature law (Rahimi & Recht, cited P:L83): for W ~ N(0, sigma^2 I),
    b ~ U[0,2pi), E[sin(Wx+b) sin(Wx'+b)] = 1/2 exp(-sigma^2 |x-x'|^2 / 2).  The paper's P:L83
    omits the 1/2."""
    d, F, sigma = 2, 200000, 3.0
    W, b = oracle.features(d, F, sigma, seed=3)
    g = np.random.default_rng(0)
    X = g.random((20, d))
    H, _ = col(W, b, X, wl.op_identity(d))          # unnormalized features, (20, F)
    K = H @ H.T / F
    r2 = ((X[:, None, :] - X[None, :, :]) ** 2).sum(-1)
    ref = 0.5 * np.exp(-sigma**2 * r2 / 2)
    assert np.abs(K - ref).max() < 0.02


# ----------------------------------------------------------------------------- symbolic cycle
def test_diff_cycle_closed_form():
    """pin: Eq. 2 in closed form: D^alpha -> (e = alpha, p = |alpha| mod 4)."""
    for d in (1, 2, 3):
        for alpha in itertools.product(range(6), repeat=d):
            e, p = oracle.diff(alpha)
            assert e == tuple(alpha)
            assert p == sum(alpha) % 4


def test_worked_values_golden():
    """pin: worked values (tests/golden/worked_values.json, each with its citation)."""
    cases = json.load(open(os.path.join(GOLDEN, "worked_values.json")))["cases"]
    for c in cases:
        W = np.array(c["W"])
        b = np.array(c["b"])
        A, _ = col(W, b, np.array([c["x"]]), [(tuple(c["alpha"]), 1.0, -1)])
        assert abs(A[0, 0] - c["value"]) <= 4e-15 * max(1.0, abs(c["value"])), c["cite"]


def test_four_step_cycle_returns():
    """pin: P:L97 / App. F P:L709 -- four derivatives return to sin, times W^4."""
    W, b = rand_basis(1, 50, 3.0, 1)
    X = np.random.default_rng(2).uniform(-1, 1, (30, 1))
    H, _ = col(W, b, X, [((0,), 1.0, -1)])
    for a in range(4):
        Da, _ = col(W, b, X, [((a,), 1.0, -1)])
        Da4, S = col(W, b, X, [((a + 4,), 1.0, -1)])
        assert np.allclose(Da4, Da * W[:, 0] ** 4, rtol=0, atol=1e-13 * S.max())


# ----------------------------------------------------------------------------- closed forms (Cor. 1)
@pytest.mark.parametrize("d", [1, 2, 3, 5])
def test_laplacian_biharmonic_helmholtz_closed_forms(d):
    """pins: Cor. 1: Lap phi = -|W|^2 phi, Lap^2 phi = |W|^4 phi; Helmholtz
    (k^2 - |W|^2) phi; phi evaluated with numpy's library sin."""
    W, b = rand_basis(d, 64, 2.0, d)
    X = np.random.default_rng(d).random((40, d))
    phi = np.sin(X @ W.T + b)                       # library routine
    w2 = (W**2).sum(1)
    L, S = col(W, b, X, wl.op_laplacian(d))
    assert np.abs(L - (-w2) * phi).max() <= 1e-13 * S.max()
    B, S = col(W, b, X, wl.op_biharmonic(d))
    assert np.abs(B - (w2**2) * phi).max() <= 1e-13 * S.max()
    k = 10.0
    Hm, S = col(W, b, X, wl.op_laplacian(d) + [(tuple([0] * d), k * k, -1)])
    assert np.abs(Hm - (k * k - w2) * phi).max() <= 1e-13 * S.max()


def test_advection_closed_form_and_quarter_wave():
    """pins: Cor. 1 advection (v.W) cos with numpy cos; App. F quarter-wave shift
    (P:L741): b -> b + pi/2 turns the sin column into the cos column."""
    d = 3
    W, b = rand_basis(d, 50, 3.0, 7)
    X = np.random.default_rng(8).random((25, d))
    v = np.array([0.3, -1.2, 2.0])
    A, S = col(W, b, X, wl.op_advection(v))
    ref = (W @ v) * np.cos(X @ W.T + b)
    assert np.abs(A - ref).max() <= 1e-13 * S.max()
    D1, S1 = col(W, b, X, wl.op_partial(d, 0, 1))
    H, _ = col(W, b + np.pi / 2, X, wl.op_identity(d))
    assert np.abs(D1 - W[:, 0] * H).max() <= 1e-13 * S1.max()


def test_identity_is_feature_matrix_and_normalization():
    """pins: identity operator gives H and the 1/sqrt(N) factor of Eq. 1."""
    d, F = 2, 37
    W, b = rand_basis(d, F, 1.5, 3)
    X = np.random.default_rng(4).random((11, d))
    H, _ = col(W, b, X, wl.op_identity(d), normalize=True)
    assert np.abs(H - np.sin(X @ W.T + b) / math.sqrt(F)).max() < 1e-15


# ----------------------------------------------------------------------------- brute force FD
def _stencil(order, h):
    c = {1: [-0.5, 0.0, 0.5], 2: [1.0, -2.0, 1.0], 3: [-0.5, 1.0, 0.0, -1.0, 0.5],
         4: [1.0, -4.0, 6.0, -4.0, 1.0]}[order]
    m = len(c) // 2
    return [((k - m) * h, ck / h**order) for k, ck in enumerate(c)]


def _fd(W, b, x, alpha, h):
    """tensor-product central difference of phi_j = sin(W_j.x + b_j) (library np.sin);
    h is the per-axis step vector"""
    per_axis = [_stencil(a, h[k]) if a > 0 else [(0.0, 1.0)] for k, a in enumerate(alpha)]
    acc = np.zeros(W.shape[0])
    for combo in itertools.product(*per_axis):
        off = np.array([o for o, _ in combo], float)
        w = np.prod([c for _, c in combo])
        acc += w * np.sin(W @ (x + off) + b)
    return acc


@pytest.mark.parametrize("d", [1, 2, 3, 5])
def test_arbitrary_alpha_vs_finite_differences(d):
    """pin: brute force -- Richardson-extrapolated central differences of the plain feature
    (AC1 S:L685), every alpha with |alpha| <= 4 (d <= 2) or a sample (d > 2)."""
    W, b = rand_basis(d, 16, 1.5, 10 + d)
    g = np.random.default_rng(d)
    alphas = [a for a in itertools.product(range(5), repeat=d) if 1 <= sum(a) <= 4]
    if len(alphas) > 40:
        alphas = [alphas[i] for i in g.choice(len(alphas), 40, replace=False)]
    for alpha in alphas:
        x = g.random(d)
        A, S = col(W, b, x[None, :], [(tuple(alpha), 1.0, -1)])
        # per-feature, per-axis step h_jk = 0.05 / |W_jk| keeps both the O(h^4) truncation and
        # the eps / prod h^alpha rounding of the stencil far below 1e-6 relative to S
        fd = np.zeros(W.shape[0])
        for j in range(W.shape[0]):
            h = 0.05 / np.maximum(np.abs(W[j]), 1e-6)
            Wj, bj = W[j:j + 1], b[j:j + 1]
            fd[j] = ((4 * _fd(Wj, bj, x, alpha, h / 2) - _fd(Wj, bj, x, alpha, h)) / 3)[0]
        err = np.abs(A[0] - fd) / S[0]
        assert err.max() <= 1e-6, (alpha, err.max())


def test_sign_and_index_errors_would_fail():
    """pin (mutation guard): the cycle sign pattern (+,+,-,-) and the per-axis exponent are
    visible -- e.g. d^3/dx^3 sin(Wx+b) = -W^3 cos(Wx+b) by calculus."""
    W = np.array([[1.7, -0.4]])
    b = np.array([0.3])
    x = np.array([[0.2, 0.9]])
    z = float(W[0] @ x[0] + b[0])
    A, _ = col(W, b, x, [((3, 0), 1.0, -1)])
    assert abs(A[0, 0] - (-(1.7**3) * math.cos(z))) < 1e-14
    A, _ = col(W, b, x, [((0, 2), 1.0, -1)])
    assert abs(A[0, 0] - (-(0.4**2) * math.sin(z))) < 1e-14
    A, _ = col(W, b, x, [((1, 1), 1.0, -1)])
    assert abs(A[0, 0] - (-(1.7 * -0.4) * math.sin(z))) < 1e-14


def test_linearity_in_the_operator():
    """pin: L -> A is linear: A(a L1 + b L2) = a A(L1) + b A(L2) to rounding"""
    from hypothesis import given, settings
    from hypothesis import strategies as st

    @settings(max_examples=25, deadline=None)
    @given(st.integers(1, 4), st.floats(-3, 3), st.floats(-3, 3), st.integers(0, 10_000))
    def check(d, ca, cb, seed):
        g = np.random.default_rng(seed)
        W, b = rand_basis(d, 17, 2.0, seed)
        X = g.random((9, d))
        L1 = [(tuple(int(v) for v in g.integers(0, 3, d)), float(g.normal()), -1) for _ in range(2)]
        L2 = [(tuple(int(v) for v in g.integers(0, 3, d)), float(g.normal()), -1) for _ in range(3)]
        A1, S1 = col(W, b, X, L1)
        A2, S2 = col(W, b, X, L2)
        A12, _ = col(W, b, X, [(a, ca * c, f) for a, c, f in L1] + [(a, cb * c, f) for a, c, f in L2])
        scale = abs(ca) * S1 + abs(cb) * S2
        assert np.all(np.abs(A12 - (ca * A1 + cb * A2)) <= 1e-13 * np.maximum(scale, 1e-300) + 1e-300)
    check()


# ----------------------------------------------------------------------------- blocks / fields
def test_row_blocks_lambda_and_rhs():
    """pins: Eq. 3 row order pde -> bc and weights on both A and b; doubling lambda
    doubles only the BC rows and their rhs."""
    p = wl.make_problem("c2_poisson2d", "mini")
    W, b = p.parity_features()
    A1, r1, _ = oracle.assemble(W, b, p.blocks)
    p.blocks[1].weight *= 2
    A2, r2, _ = oracle.assemble(W, b, p.blocks)
    n0 = p.blocks[0].n
    assert np.array_equal(A1[:n0], A2[:n0]) and np.array_equal(r1[:n0], r2[:n0])
    assert np.array_equal(2 * A1[n0:], A2[n0:]) and np.array_equal(2 * r1[n0:], r2[n0:])
    assert np.array_equal(r1[:n0], p.blocks[0].values)
    # arbitrary row subsets equal the corresponding rows of the full assembly
    rows = np.array([n0 + 3, 0, 7, n0 - 1, n0])
    As, rs, _ = oracle.assemble(W, b, p.blocks, rows=rows)
    assert np.array_equal(As, A2[rows]) and np.array_equal(rs, r2[rows])


def test_coefficient_field_term():
    """pin: variable coefficient c(x) multiplies its term per point."""
    d = 3
    W, b = rand_basis(d, 20, 2.0, 5)
    X = np.random.default_rng(6).random((9, d))
    c = 1.0 + X[:, 0]
    A, _ = col(W, b, X, [((0, 0, 0), 16.0, 0)], fields=c[:, None])
    ref = 16.0 * c[:, None] * np.sin(X @ W.T + b)
    assert np.abs(A - ref).max() < 1e-12


# ----------------------------------------------------------------------------- least squares
def test_lstsq_identity_and_library_agreement():
    """pins: A = I -> beta = b; full-rank random systems agree with LAPACK
    (numpy.linalg.lstsq) and satisfy the normal equations."""
    n = 12
    bv = np.arange(n, dtype=float) - 3.5
    beta, res, _ = oracle.lstsq(np.eye(n), bv)
    assert np.allclose(beta, bv, atol=1e-15) and res < 1e-14
    g = np.random.default_rng(0)
    for m, n in [(50, 10), (200, 37), (37, 37)]:
        A = g.normal(size=(m, n))
        bv = g.normal(size=m)
        beta, res, _ = oracle.lstsq(A, bv)
        ref, *_ = np.linalg.lstsq(A, bv, rcond=None)
        assert np.abs(beta - ref).max() <= 1e-10 * max(1, np.abs(ref).max())
        ne = A.T @ (A @ beta - bv)
        assert np.linalg.norm(ne) <= 1e-10 * np.linalg.norm(A.T @ bv)
        assert abs(res - np.linalg.norm(A @ beta - bv)) <= 1e-10 * max(1, res)


def test_lstsq_ridge_matches_stacked_library():
    """pin: Tikhonov form == plain lstsq of [A; sqrt(mu) I] (LAPACK), sqrt(mu) =
    tau ||A||_F (reading A16); mu = 0 reduces to lstsq."""
    g = np.random.default_rng(1)
    A = g.normal(size=(60, 20))
    A[:, 5] = A[:, 4]                                  # rank deficient
    bv = g.normal(size=60)
    tau = 1e-3
    beta, _, _ = oracle.lstsq(A, bv, ridge_rel=tau)
    sq = tau * np.linalg.norm(A)
    ref, *_ = np.linalg.lstsq(np.vstack([A, sq * np.eye(20)]), np.concatenate([bv, np.zeros(20)]),
                              rcond=None)
    assert np.abs(beta - ref).max() <= 1e-9 * np.abs(ref).max()


def test_lstsq_zero_column_raises():
    A = np.ones((5, 3))
    A[:, 1] = 0
    with pytest.raises(np.linalg.LinAlgError):
        oracle.lstsq(A, np.ones(5))


# ----------------------------------------------------------------------------- eval
def test_eval_unit_coefficient_reproduces_feature():
    """pins: beta = sqrt(N) e_j -> u = phi_j exactly; beta = 0 -> 0."""
    d, F = 3, 25
    W, b = rand_basis(d, F, 2.0, 9)
    X = np.random.default_rng(1).random((30, d))
    for j in (0, 7, 24):
        beta = np.zeros(F)
        beta[j] = math.sqrt(F)
        u = oracle.evaluate(W, b, beta, X)
        assert np.abs(u - np.sin(X @ W[j] + b[j])).max() < 1e-15
    assert np.all(oracle.evaluate(W, b, np.zeros(F), X) == 0)


# ----------------------------------------------------------------------------- manufactured recovery
def test_spec_poisson_1d_recovery():
    """pin: closed-form u* -- -u'' = pi^2 sin(pi x), u(0)=u(1)=0, N=200, M=1000 -> rel L2 <= 1e-6
    (AC3 S:L687)."""
    g = np.random.default_rng(0)
    Xi = g.random((1000, 1))
    Xb = np.array([[0.0], [1.0]])
    W = g.normal(0, 3.0, (200, 1))
    b = g.uniform(0, 2 * np.pi, 200)
    blocks = [Blk(Xi, wl.op_laplacian(1, -1.0), 1.0, np.pi**2 * np.sin(np.pi * Xi[:, 0])),
              Blk(Xb, wl.op_identity(1), 100.0, np.zeros(2))]
    A, rhs, _ = oracle.assemble(W, b, blocks)
    beta, _, _ = oracle.lstsq(A, rhs)
    Xt = np.linspace(0, 1, 501)[:, None]
    u = oracle.evaluate(W, b, beta, Xt)
    ref = np.sin(np.pi * Xt[:, 0])
    assert np.linalg.norm(u - ref) / np.linalg.norm(ref) <= 1e-6


@pytest.mark.parametrize("name,tol", [("c1_poisson1d", 1e-9), ("c2_poisson2d", 1e-6),
                                      ("c4_heat2d", 1e-4)])
def test_config_recovery(name, tol):
    """pin: manufactured u* of BASELINE configs (C1 full size; C2/C4 reduced) recovered by
    oracle assemble -> lstsq -> eval at held-out points."""
    p = wl.make_problem(name, "full" if name == "c1_poisson1d" else "mini")
    W, b = p.parity_features()
    A, rhs, _ = oracle.assemble(W, b, p.blocks)
    beta, _, _ = oracle.lstsq(A, rhs, ridge_rel=p.ridge_rel)
    Xt = p.test_points(2000)
    u = oracle.evaluate(W, b, beta, Xt)
    us = p.u_star(Xt)
    assert np.linalg.norm(u - us) / np.linalg.norm(us) <= tol


# ----------------------------------------------------------------------------- SPEC identities
def test_zero_phase_rows():
    """pin: at zero phase (x = 0, b = 0) the identity row is sin(0) = 0 and a
    first-derivative row is W_j cos(0) = W_j (scaled by s = 1/sqrt(N))."""
    d, F = 2, 9
    W, _ = rand_basis(d, F, 2.0, 11)
    b = np.zeros(F)
    X = np.zeros((1, d))
    H, _ = col(W, b, X, wl.op_identity(d), normalize=True)
    assert np.all(H == 0.0)
    Dx, _ = col(W, b, X, [((1, 0), 1.0, -1)], normalize=True)
    assert np.allclose(Dx[0], W[:, 0] / math.sqrt(F), rtol=1e-15, atol=0)


def test_axis_permutation_symmetry():
    """pin: permuting the coordinate axes of X, W and every multi-index together
    leaves A unchanged, exactly (same products in the same order up to commutation)."""
    d, F = 3, 23
    W, b = rand_basis(d, F, 2.0, 12)
    X = np.random.default_rng(13).random((17, d))
    terms = [((2, 1, 0), 1.5, -1), ((0, 0, 3), -0.25, -1), ((1, 0, 1), 2.0, -1)]
    perm = [2, 0, 1]
    A, _ = col(W, b, X, terms)
    tp = [(tuple(a[p] for p in perm), c, f) for a, c, f in terms]
    Ap, _ = col(W[:, perm], b, X[:, perm], tp)
    assert np.allclose(A, Ap, rtol=1e-14, atol=1e-14 * np.abs(A).max())


def test_zero_source_gives_zero_beta_and_mu0_is_lstsq():
    """pins: a zero right-hand side gives beta = 0 exactly (Q^T 0 = 0); the Tikhonov
    solve with mu = 0 is the plain least-squares solve."""
    g = np.random.default_rng(14)
    A = g.normal(size=(40, 12))
    beta, res, _ = oracle.lstsq(A, np.zeros(40))
    assert np.all(beta == 0.0) and res == 0.0
    bv = g.normal(size=40)
    b1, r1, _ = oracle.lstsq(A, bv)
    b2, r2, _ = oracle.lstsq_mu(A, bv, 0.0)
    assert np.allclose(b1, b2, rtol=1e-13, atol=1e-13) and abs(r1 - r2) <= 1e-13 * max(r1, 1.0)


# ------------------------------------------------------------------------------------------------
# Alg. 1 line 2 ("Sample collocation points"): orc_sample_box / orc_sample_faces.
# Pinned to numpy's own Philox4x64-10 (library routine of the same generator) with the uniform map
# of DESIGN.md R1, u = (raw >> 11) 2^-53, written here independently of the oracle, plus the
# geometric facts every sample must satisfy (face counts and order, on-face coordinates, in-box,
# per-axis uniformity).
# ------------------------------------------------------------------------------------------------
def _np_uniform(seed, stream, n):
    raw = np.random.Philox(key=seed + (stream << 64)).random_raw(n)
    return (raw >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


@pytest.mark.parametrize("dim,n,seed,stream", [(1, 7, 0, 3), (2, 33, 0, 3), (3, 101, 5, 6),
                                               (5, 64, 0, 3), (8, 9, 2 ** 40 + 3, 11)])
def test_sample_box_matches_numpy_philox(dim, n, seed, stream):
    """pin: X[i][k] = lo_k + (hi_k - lo_k) u(i*dim + k) -- row-major word order, the stream's
    key word, the 53-bit uniform and the affine map, each checked bit-exactly against numpy"""
    g = np.random.default_rng(dim * 1000 + n)
    lo = g.uniform(-2.0, 0.5, dim)
    hi = lo + g.uniform(0.25, 3.0, dim)
    X = oracle.sample_box(dim, n, lo, hi, seed, stream)
    assert X.shape == (n, dim)
    u = _np_uniform(seed, stream, n * dim).reshape(n, dim)
    ref = lo[None, :] + (hi - lo)[None, :] * u          # numpy: no contraction, same rounding
    assert np.array_equal(X, ref)
    # the transposed word order (k * n + i) is a different array: the pin would catch it
    if n > 1 and dim > 1:
        wrong = lo[None, :] + (hi - lo)[None, :] * u.reshape(dim, n).T
        assert not np.array_equal(X, wrong)
    # another stream is another array (the stream is the key's high word)
    assert not np.array_equal(X, oracle.sample_box(dim, n, lo, hi, seed, stream + 1))
    assert np.all(X >= lo) and np.all(X < hi)


@pytest.mark.parametrize("dim,per_face,mask", [(2, 5, 0b11), (3, 4, 0b011), (5, 3, 0b11111),
                                               (3, 6, 0b101), (1, 2, 0b1)])
def test_sample_faces_matches_numpy_philox_and_geometry(dim, per_face, mask):
    """pin: for each axis k in the mask (increasing k): per_face points on x_k = lo_k, then
    per_face on x_k = hi_k; the other coordinates are word row*dim + l of the stream mapped to
    [lo_l, hi_l).  Checked against numpy's Philox and the face geometry"""
    lo = np.linspace(-1.0, 0.0, dim)
    hi = lo + np.linspace(1.0, 2.0, dim)
    seed, stream = 0, 4
    X = oracle.sample_faces(dim, per_face, mask, lo, hi, seed, stream)
    axes = [k for k in range(dim) if mask & (1 << k)]
    rows = 2 * per_face * len(axes)
    assert X.shape == (rows, dim)
    u = _np_uniform(seed, stream, rows * dim).reshape(rows, dim)
    ref = lo[None, :] + (hi - lo)[None, :] * u
    r = 0
    for k in axes:
        for side, val in ((0, lo[k]), (1, hi[k])):
            blk = X[r:r + per_face]
            assert np.all(blk[:, k] == val), f"face {k}/{side}: coordinate not pinned to the face"
            others = [l for l in range(dim) if l != k]
            assert np.array_equal(blk[:, others], ref[r:r + per_face, others])
            r += per_face
    assert r == rows
    assert np.all(X >= lo) and np.all(X <= hi)


def test_sample_box_uniform_ks_per_axis():
    """statistical pin: every axis of the box sample is U[lo_k, hi_k) (KS, p > 1e-4), and the
    axes are uncorrelated"""
    dim, n = 5, 20_000
    lo = np.array([0.0, -1.0, 2.0, 0.0, -3.0])
    hi = np.array([1.0, 1.0, 2.5, 10.0, -2.0])
    X = oracle.sample_box(dim, n, lo, hi, 0, 3)
    for k in range(dim):
        assert stats.kstest(X[:, k], "uniform", args=(lo[k], hi[k] - lo[k])).pvalue > 1e-4
    Cm = np.corrcoef(X.T)
    assert np.max(np.abs(Cm - np.eye(dim))) < 5.0 / math.sqrt(n)


# ----------------------------------------------------------------------------- truth mode
def _mp_deriv(Wj, bj, x, alpha):
    """D^alpha sin(W_j.x + b_j) at x by mpmath's numerical differentiation (40 digits): an
    independent brute-force value, no derivative cycle involved"""
    import mpmath as mp
    d = len(x)
    f = lambda *xs: mp.sin(mp.fsum(mp.mpf(float(Wj[k])) * xs[k] for k in range(d)) + mp.mpf(float(bj)))
    pt = tuple(mp.mpf(float(v)) for v in x)
    if sum(alpha) == 0:
        return f(*pt)
    return mp.diff(f, pt, tuple(int(a) for a in alpha))


@pytest.mark.parametrize("d", [1, 2, 3])
def test_truth_mode_matches_mpmath_derivatives(d):
    """pin: the long-double 'truth' assembly equals mpmath's 40-digit
    numerical derivatives of the plain feature to the final rounding to double (<= 2 ulp of
    the A14 scale), for every alpha with |alpha| <= 4 (a sample for d = 3), several points"""
    import mpmath as mp
    mp.mp.dps = 40
    W, b = rand_basis(d, 5, 3.0, 40 + d)
    g = np.random.default_rng(100 + d)
    alphas = [a for a in itertools.product(range(5), repeat=d) if sum(a) <= 4]
    if len(alphas) > 16:
        alphas = [alphas[i] for i in g.choice(len(alphas), 16, replace=False)]
    for alpha in alphas:
        X = g.random((2, d))
        terms = [(tuple(alpha), 1.0, -1)]
        At = oracle.assemble_truth(W, b, [Blk(X, terms)], normalize=False)
        _, S = col(W, b, X, terms)
        for i in range(X.shape[0]):
            for j in range(W.shape[0]):
                ref = _mp_deriv(W[j], b[j], X[i], alpha)
                err = abs(mp.mpf(float(At[i, j])) - ref) / mp.mpf(float(S[i, j]))
                assert err <= 3e-16, (alpha, i, j, float(err))


def test_fp64_oracle_error_against_truth():
    """the fp64 oracle's own error on the configs' operators, measured against truth mode: it
    stays ~1e-15 of the A14 scale at the configs' phase range -- far below the 1e-12 parity
    bar, so the oracle is a sound reference for the GPU path"""
    worst = 0.0
    for name in wl.CONFIG_NAMES:
        p = wl.make_problem(name, "mini")
        W, b = p.parity_features()
        R = p.n_rows
        rows = np.linspace(0, R - 1, 12).astype(np.int64)
        A, _, S = oracle.assemble(W, b, p.blocks, rows=rows)
        At = oracle.assemble_truth(W, b, p.blocks, rows=rows)
        e = float((np.abs(A - At) / S).max())
        worst = max(worst, e)
        assert e <= 2e-14, (name, e)
    assert worst > 0.0   # the two differ (fp64 vs long double): the comparison is not vacuous
