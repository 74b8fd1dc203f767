"""GPU parity: libfls (through the C ABI) against the CPU oracle, element by element.

Entry metric: |A_gpu - A_orc| <= 1e-12 * S_ij with
S_ij = w s sum_t |c_t(x_i)| |prod_k W_jk^alpha_tk|.  rhs entries are a single product on both
sides and must be bit-exact.  Fitted u at 10,000 held-out points: relative L2 <= 1e-6.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import workloads as wl
from gpu_common import ENTRY_TOL, U_TOL, dev_blocks, rows_from_colmajor, scaled_err

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2602_10541_b200 import fls


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return fls.Context()


def _parity_feats(p):
    W, b = p.parity_features()
    return W, b, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda()


# ------------------------------------------------------------------------------------- a1
@pytest.mark.parametrize("dim,F,sigma,seed", [(1, 500, 10.0, 0), (3, 8192, 3.0, 0),
                                              (5, 4001, 2.0, 7), (2, 1, 5.0, 2**64 - 1)])
def test_features_match_oracle(ctx, dim, F, sigma, seed):
    Wd, bd = fls.fls_features(ctx, dim, F, sigma, seed)
    fls.fls_sync(ctx)
    Wo, bo = oracle.features(dim, F, sigma, seed)
    assert np.array_equal(bd.cpu().numpy(), bo)                 # one correctly rounded product
    Wg = Wd.cpu().numpy()
    ulp = np.spacing(np.abs(Wo))
    assert np.all(np.abs(Wg - Wo) <= 8 * ulp + 1e-300), np.max(np.abs(Wg - Wo) / ulp)
    Wd2, bd2 = fls.fls_features(ctx, dim, F, sigma, seed)
    assert torch.equal(Wd, Wd2) and torch.equal(bd, bd2)


# ------------------------------------------------------------------------------------- a2-a8
@pytest.mark.parametrize("name", wl.CONFIG_NAMES)
def test_assemble_parity_mini(ctx, name):
    p = wl.make_problem(name, "mini")
    W, b, Wd, bd = _parity_feats(p)
    F = p.n_features
    Ab, lda = fls.fls_assemble(ctx, Wd, bd, dev_blocks(p))
    fls.fls_sync(ctx)
    Ao, ro, S = oracle.assemble(W, b, p.blocks)
    Ag, rg = rows_from_colmajor(Ab, lda, F, np.arange(p.n_rows))
    emax, e999 = scaled_err(Ag, Ao, S)
    assert emax <= ENTRY_TOL, (emax, e999)
    assert np.array_equal(rg, ro)


@pytest.mark.parametrize("name", ["c2_poisson2d", "c3_poisson5d", "c4_heat2d", "c5_biharm3d"])
def test_assemble_parity_full_size_sampled_rows(ctx, name):
    """BASELINE.json full sizes in the bench's launch configuration, oracle on sampled rows."""
    p = wl.make_problem(name, "full")
    F, R = p.n_features, p.n_rows
    need = (F + 1) * wl_round4(R) * 8
    free, _ = torch.cuda.mem_get_info()
    if need + (2 << 30) > free:
        pytest.skip(f"needs {need / 1e9:.1f} GB, {free / 1e9:.1f} GB free")
    W, b, Wd, bd = _parity_feats(p)
    Ab, lda = fls.fls_assemble(ctx, Wd, bd, dev_blocks(p))
    fls.fls_sync(ctx)
    rows = wl.sample_rows(R, 8, 256 if R > 100_000 else 61)
    Ag, rg = rows_from_colmajor(Ab, lda, F, rows)
    del Ab
    torch.cuda.empty_cache()
    Ao, ro, S = oracle.assemble(W, b, p.blocks, rows=rows)
    emax, e999 = scaled_err(Ag, Ao, S)
    assert emax <= ENTRY_TOL, (emax, e999)
    assert np.array_equal(rg, ro)


@pytest.mark.parametrize("name", ["c3_poisson5d", "c5_biharm3d"])
def test_bench_call_full_size_vs_oracle(ctx, name):
    """bench.py's exact call (fls_features_assemble: W, b drawn on the device from the seed,
    full BASELINE size, the bench's lda) against the oracle given ITS OWN features
    (oracle.features, same seed) on sampled rows: W may differ by <= 8 ulp, which moves an
    entry by well under the A14 bound."""
    p = wl.make_problem(name, "full")
    F, R, d = p.n_features, p.n_rows, p.dim
    lda = wl_round4(R)
    need = (F + 1) * lda * 8
    free, _ = torch.cuda.mem_get_info()
    if need + (2 << 30) > free:
        pytest.skip(f"needs {need / 1e9:.1f} GB, {free / 1e9:.1f} GB free")
    Ab = torch.empty(((F + 1) * lda,), dtype=torch.float64, device="cuda")
    W = torch.empty((F, d), dtype=torch.float64, device="cuda")
    b = torch.empty((F,), dtype=torch.float64, device="cuda")
    bset = fls.BlockSet(dev_blocks(p), d)
    fls.fls_features_assemble(ctx, d, F, p.sigma, p.seed, bset, W=W, b=b, A=Ab, lda=lda)
    fls.fls_sync(ctx)
    rows = wl.sample_rows(R, 8, 256 if R > 100_000 else 61)
    Ag, rg = rows_from_colmajor(Ab, lda, F, rows)
    del Ab
    torch.cuda.empty_cache()
    Wo, bo = oracle.features(d, F, float(p.sigma), int(p.seed))
    Ao, ro, S = oracle.assemble(Wo, bo, p.blocks, rows=rows)
    emax, e999 = scaled_err(Ag, Ao, S)
    assert emax <= ENTRY_TOL, (emax, e999)
    assert np.array_equal(rg, ro)


def wl_round4(n):
    return ((n + 3) // 4) * 4


# ------------------------------------------------------------------------------------- layouts, shards
def test_row_major_and_shards_bit_identical(ctx):
    p = wl.make_problem("c4_heat2d", "mini")
    _, _, Wd, bd = _parity_feats(p)
    F, R = p.n_features, p.n_rows
    blocks = fls.BlockSet(dev_blocks(p), 3)
    Ab, lda = fls.fls_assemble(ctx, Wd, bd, blocks)
    full = Ab[: (F + 1) * lda].view(F + 1, lda)[:, :R].T.contiguous()   # (R, F+1)
    Arm, rrm = fls.fls_assemble(ctx, Wd, bd, blocks, layout=fls.FLS_ROW_MAJOR)
    assert torch.equal(Arm[:, :F], full[:, :F]) and torch.equal(rrm, full[:, F])
    for P in (2, 3, 8):
        for r in range(P):
            a, e = wl.shard_range(R, r, P)
            Ash, ldl = fls.fls_assemble(ctx, Wd, bd, blocks, row_begin=a, row_end=e)
            sh = Ash[: (F + 1) * ldl].view(F + 1, ldl)[:, : e - a].T
            assert torch.equal(sh, full[a:e]), (P, r)
    fls.fls_sync(ctx)


def test_row_major_multi_chunk_staging(ctx):
    """row-major CTAs that stage several 64-row chunks of points (double-buffered cp.async)
    with a ragged last chunk, a coefficient field (G = 1), an odd feature count (the last
    thread's second feature is out of range) and a block starting at an odd row: bit-identical
    to the column-major layout, sampled rows within the entry tolerance of the oracle"""
    d, F = 3, 101
    g = np.random.default_rng(7)
    W = g.normal(0, 3, (F, d))
    b = g.uniform(0, 2 * math.pi, F)
    Wd, bd = torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda()
    sizes = [299_999, 1_003]
    terms = wl.op_biharmonic(3) + [((0, 0, 0), 16.0, 0)]
    Xs = [g.random((n, d)) for n in sizes]
    fs = [1.0 + g.random((n, 1)) for n in sizes]
    vals = [g.random(n) for n in sizes]
    blocks = [fls.Block(torch.from_numpy(X).cuda(), terms, w, torch.from_numpy(v).cuda(),
                        torch.from_numpy(f).cuda()) for X, v, f, w in zip(Xs, vals, fs, (1.0, 3.0))]
    R = sum(sizes)
    Ab, lda = fls.fls_assemble(ctx, Wd, bd, blocks)
    Arm, rrm = fls.fls_assemble(ctx, Wd, bd, blocks, layout=fls.FLS_ROW_MAJOR)
    fls.fls_sync(ctx)
    full = Ab[: (F + 1) * lda].view(F + 1, lda)[:, :R]
    assert torch.equal(Arm[:, :F], full[:F].T) and torch.equal(rrm, full[F])

    class B:
        def __init__(s, X, v, f, w):
            s.X, s.terms, s.weight, s.values, s.fields = X, terms, w, v, f
    rows = np.unique(np.concatenate([np.linspace(0, R - 1, 97).astype(np.int64),
                                     np.arange(299_990, 300_010)]))
    Ao, ro, S = oracle.assemble(W, b, [B(X, v, f, w) for X, v, f, w in zip(Xs, vals, fs, (1.0, 3.0))],
                                rows=rows)
    Mr = Arm[torch.from_numpy(rows).cuda()].cpu().numpy()
    assert scaled_err(Mr[:, :F], Ao, S)[0] <= ENTRY_TOL
    assert np.array_equal(rrm.cpu().numpy()[rows], ro)


def test_user_stream_and_timing_hook(ctx):
    """a ctx on a user stream produces the same entries; the timing hook counts the assembly
    launches (one per batch of blocks sharing a kernel variant) and resets on read"""
    p = wl.make_problem("c4_heat2d", "mini")
    _, _, Wd, bd = _parity_feats(p)
    blocks = fls.BlockSet(dev_blocks(p), 3)
    ref, lda = fls.fls_assemble(ctx, Wd, bd, blocks)
    fls.fls_sync(ctx)
    s = torch.cuda.Stream()
    c2 = fls.Context(stream=s)
    with torch.cuda.stream(s):
        fls.fls_ctx_timing(c2, True)
        got, _ = fls.fls_assemble(c2, Wd, bd, blocks)
        fls.fls_assemble(c2, Wd, bd, blocks, A=got, lda=lda)
        ms, n = fls.fls_ctx_timing_read(c2)
        ms2, n2 = fls.fls_ctx_timing_read(c2)
    fls.fls_sync(c2)
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
    assert n == 2 and ms > 0 and n2 == 0          # pde + bc + ic share one variant -> 1 launch/call
    c2.close()


def test_set_stream_orders_pending_work(ctx):
    """fls_ctx_set_stream: work enqueued on the old stream completes before the ctx's next call
    on the new stream runs (include/fls.h) -- here the old stream is held up by a ~50 ms spin
    before the assembly, and fls_frob2 on the new stream must still see the assembled A"""
    p = wl.make_problem("c4_heat2d", "mini")
    _, _, Wd, bd = _parity_feats(p)
    blocks = fls.BlockSet(dev_blocks(p), 3)
    ref, lda = fls.fls_assemble(ctx, Wd, bd, blocks)
    fls.fls_sync(ctx)
    F = p.n_features
    want = float((ref.reshape(-1)[:F * lda].view(F, lda)[:, :p.n_rows] ** 2).sum())
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    A = torch.zeros_like(ref)
    torch.cuda.synchronize()
    c2 = fls.Context(stream=s1)
    with torch.cuda.stream(s1):
        torch.cuda._sleep(100_000_000)             # ~50 ms at 1.9 GHz on s1 only
    fls.fls_assemble(c2, Wd, bd, blocks, A=A, lda=lda)
    c2.set_stream(s2)
    got = fls.fls_frob2(c2, A, p.n_rows, lda, F)
    torch.cuda.synchronize()
    assert got == pytest.approx(want, rel=1e-12)
    c2.close()


def test_unaligned_lda_and_pointer_scalar_path(ctx):
    p = wl.make_problem("c2_poisson2d", "mini")
    _, _, Wd, bd = _parity_feats(p)
    F, R = p.n_features, p.n_rows
    blocks = fls.BlockSet(dev_blocks(p), 2)
    Ab, lda = fls.fls_assemble(ctx, Wd, bd, blocks)
    ref = Ab[: (F + 1) * lda].view(F + 1, lda)[:, :R]
    lda2 = R + 1                                    # odd lda -> scalar stores
    buf = torch.full(((F + 1) * lda2 + 1,), float("nan"), dtype=torch.float64, device="cuda")
    A2 = buf[1:]                                    # 8-byte (not 16-byte) aligned
    fls.fls_assemble(ctx, Wd, bd, blocks, A=A2, lda=lda2)
    got = A2[: (F + 1) * lda2].view(F + 1, lda2)[:, :R]
    assert torch.equal(got, ref)
    assert torch.isnan(A2[lda2 - 1])                # padding row untouched


@pytest.mark.parametrize("d", [1, 2, 3, 5])
def test_point_loads_vector_and_scalar_paths(ctx, d):
    """the CTA prologue loads a row pair's points (and a single coefficient field) as 16-byte
    vectors when the pair starts on a 16-byte boundary, else element by element: blocks that
    start at odd rows, X / field arrays 8 bytes off a 16-byte boundary and a ragged tail give
    bit-identical entries to the aligned layout and match the oracle"""
    F = 37
    g = np.random.default_rng(d)
    W = g.normal(0, 2, (F, d))
    b = g.uniform(0, 2 * math.pi, F)
    Wd, bd = torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda()
    sizes = [3, 1030, 517]                       # blocks start at rows 0, 3 (odd), 1033 (odd)
    Xs = [g.random((n, d)) for n in sizes]
    fs = [1.0 + g.random((n, 1)) for n in sizes]
    vals = [g.random(n) for n in sizes]
    terms = [((2,) + (0,) * (d - 1), -1.0, -1), ((0,) * d, 4.0, 0)]   # -u_xx + 4 c(x) u

    def dev(t, off):
        """contiguous device copy whose data pointer is `off` doubles past a 16-byte boundary"""
        flat = torch.empty(t.size + 2, dtype=torch.float64, device="cuda")
        v = flat[off: off + t.size]
        v.copy_(torch.from_numpy(np.ascontiguousarray(t).ravel()))
        return v.view(t.shape)

    outs = []
    for off in (0, 1):
        blocks = [fls.Block(dev(X, off), terms, 1.0, dev(v, off), dev(f, off))
                  for X, v, f in zip(Xs, vals, fs)]
        Ab, lda = fls.fls_assemble(ctx, Wd, bd, blocks)
        fls.fls_sync(ctx)
        R = sum(sizes)
        outs.append(Ab[: (F + 1) * lda].view(F + 1, lda)[:, :R].clone())
    assert torch.equal(outs[0], outs[1])

    class B:
        def __init__(s, X, v, f):
            s.X, s.terms, s.weight, s.values, s.fields = X, terms, 1.0, v, f
    Ao, ro, S = oracle.assemble(W, b, [B(X, v, f) for X, v, f in zip(Xs, vals, fs)])
    M = outs[0].cpu().numpy()
    assert scaled_err(M[:F].T, Ao, S)[0] <= ENTRY_TOL
    assert np.array_equal(M[F], ro)


def test_empty_and_ragged_blocks(ctx):
    d, F = 3, 131
    g = np.random.default_rng(0)
    W = g.normal(0, 2, (F, d))
    b = g.uniform(0, 2 * math.pi, F)
    X1 = g.random((3, d))
    X2 = g.random((1025, d))
    Wd, bd = torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda()

    class B:
        def __init__(s, X, terms, w):
            s.X, s.terms, s.weight, s.values, s.fields = X, terms, w, np.ones(len(X)), None
    lap = wl.op_laplacian(d, -1.0)
    host = [B(np.zeros((0, d)), lap, 1.0), B(X1, lap, 1.0), B(X2, wl.op_identity(d), 7.0)]
    dev = [fls.Block(torch.from_numpy(np.ascontiguousarray(h.X)).cuda(), h.terms, h.weight,
                     torch.from_numpy(h.values).cuda()) for h in host]
    Ab, lda = fls.fls_assemble(ctx, Wd, bd, dev)
    fls.fls_sync(ctx)
    Ao, ro, S = oracle.assemble(W, b, host)
    Ag, rg = rows_from_colmajor(Ab, lda, F, np.arange(1028))
    assert scaled_err(Ag, Ao, S)[0] <= ENTRY_TOL and np.array_equal(rg, ro)
    # empty range is a no-op
    fls.fls_assemble(ctx, Wd, bd, dev, row_begin=5, row_end=5)


# ------------------------------------------------------------------------------------- operator modes
def _mode_case(ctx, terms, fields=None, d=3, F=203, n=777, seed=3):
    g = np.random.default_rng(seed)
    W = g.normal(0, 2.5, (F, d))
    b = g.uniform(0, 2 * math.pi, F)
    X = g.random((n, d))

    class B:
        pass
    h = B()
    h.X, h.terms, h.weight, h.values, h.fields = X, terms, 3.0, g.normal(size=n), fields
    dv = fls.Block(torch.from_numpy(X).cuda(), terms, 3.0, torch.from_numpy(h.values).cuda(),
                   torch.from_numpy(fields).cuda() if fields is not None else None)
    Ab, lda = fls.fls_assemble(ctx, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(), [dv])
    fls.fls_sync(ctx)
    Ao, ro, S = oracle.assemble(W, b, [h])
    Ag, rg = rows_from_colmajor(Ab, lda, F, np.arange(n))
    emax, _ = scaled_err(Ag, Ao, S)
    assert emax <= ENTRY_TOL, emax
    assert np.array_equal(rg, ro)


@pytest.mark.parametrize("d,G,mixed", [(1, 0, False), (3, 1, False), (3, 2, True), (5, 0, True),
                                       (8, 4, True)])
def test_no_out_of_bounds_writes(ctx, d, G, mixed):
    """bounds guard (compute-sanitizer is closed on this pool): NaN sentinels before A, in the
    lda padding rows and after the last column stay untouched for every kernel family, with
    ragged row ranges that start and end mid-pair and mid-tile."""
    g = np.random.default_rng(d * 10 + G)
    F, n = 261, 2051
    W = torch.from_numpy(g.normal(0, 2, (F, d))).cuda()
    b = torch.from_numpy(g.uniform(0, 6.28, F)).cuda()
    X = torch.from_numpy(g.random((n, d))).cuda()
    fields = torch.from_numpy(g.normal(size=(n, max(G, 1)))).cuda() if G else None
    terms = [(tuple([2 if k == 0 else 0 for k in range(d)]), -1.0, -1)]
    if mixed:
        terms.append((tuple([1 if k == d - 1 else 0 for k in range(d)]), 0.7, -1))
    for q in range(G):
        terms.append((tuple([0] * d), 1.0 + q, q))
    blk = [fls.Block(X, terms, 1.0, torch.ones(n, dtype=torch.float64, device="cuda"), fields)]
    for (r0, r1) in [(0, n), (1, n - 3), (513, 1500)]:
        m = r1 - r0
        lda = m + 5
        guard = 4096
        buf = torch.full((guard + (F + 1) * lda + guard,), float("nan"), dtype=torch.float64,
                         device="cuda")
        A = buf[guard: guard + (F + 1) * lda]
        fls.fls_assemble(ctx, W, b, blk, row_begin=r0, row_end=r1, A=A, lda=lda)
        fls.fls_sync(ctx)
        assert torch.isnan(buf[:guard]).all() and torch.isnan(buf[-guard:]).all()
        V = A.view(F + 1, lda)
        assert torch.isnan(V[:, m:]).all()
        assert not torch.isnan(V[:, :m]).any()


@pytest.mark.parametrize("fuse", ["0", "1000000000000"])
@pytest.mark.parametrize("d,G", [(1, 0), (3, 1), (5, 0), (8, 1)])
def test_no_out_of_bounds_writes_features_assemble(ctx, d, G, fuse, monkeypatch):
    """the same sentinel guard for fls_features_assemble, whose draws write W and b too -- the
    two-launch path (feature / prefactor kernel under PDL, then the assembly) and the ONE-launch
    path (the assembly CTAs draw, fold and write W, b themselves)"""
    monkeypatch.setenv("FLS_FUSE_MAX_ENTRIES", fuse)
    g = np.random.default_rng(d * 10 + G + 7)
    F, n = 261, 2051
    X = torch.from_numpy(g.random((n, d))).cuda()
    fields = torch.from_numpy(g.normal(size=(n, max(G, 1)))).cuda() if G else None
    terms = [(tuple([2 if k == 0 else 0 for k in range(d)]), -1.0, -1)]
    for q in range(G):
        terms.append((tuple([0] * d), 1.0 + q, q))
    blk = [fls.Block(X, terms, 1.0, torch.ones(n, dtype=torch.float64, device="cuda"), fields)]
    guard = 4096
    for (r0, r1) in [(0, n), (1, n - 3), (513, 1500)]:
        m = r1 - r0
        lda = m + 5
        buf = torch.full((guard + (F + 1) * lda + guard,), float("nan"), dtype=torch.float64,
                         device="cuda")
        wbuf = torch.full((guard + F * d + guard,), float("nan"), dtype=torch.float64, device="cuda")
        bbuf = torch.full((guard + F + guard,), float("nan"), dtype=torch.float64, device="cuda")
        A, W, b = buf[guard: -guard], wbuf[guard: -guard].view(F, d), bbuf[guard: -guard]
        fls.fls_features_assemble(ctx, d, F, 2.0, 5, blk, W=W, b=b, row_begin=r0, row_end=r1, A=A,
                                  lda=lda)
        fls.fls_sync(ctx)
        for bb in (buf, wbuf, bbuf):
            assert torch.isnan(bb[:guard]).all() and torch.isnan(bb[-guard:]).all()
        assert not torch.isnan(W).any() and not torch.isnan(b).any()
        V = A.view(F + 1, lda)
        assert torch.isnan(V[:, m:]).all()
        assert not torch.isnan(V[:, :m]).any()


def test_mode_cos_only_shift(ctx):
    _mode_case(ctx, wl.op_advection([0.5, -1.0, 2.0]))               # all odd orders


def test_mode_fold_mixed_constant(ctx):
    _mode_case(ctx, wl.op_partial(3, 2, 1) + wl.op_laplacian(3, -0.1, [0, 1])
               + [((1, 1, 1), 0.3, -1), ((0, 0, 0), 5.0, -1)])


def test_mode_sincos_with_fields(ctx):
    g = np.random.default_rng(1)
    fields = np.ascontiguousarray(g.normal(size=(777, 3)))
    terms = (wl.op_laplacian(3, 1.0) + [((1, 0, 0), 2.0, 0), ((0, 0, 0), -1.0, 2),
                                        ((0, 3, 0), 0.5, 1)])
    _mode_case(ctx, terms, fields)


def test_mode_sin_two_fields_high_order(ctx):
    g = np.random.default_rng(2)
    fields = np.ascontiguousarray(g.normal(size=(777, 2)))
    terms = wl.op_biharmonic(3) + [((0, 0, 0), 16.0, 0), ((2, 0, 0), 1.5, 1), ((0, 0, 6), 1e-3, -1)]
    _mode_case(ctx, terms, fields)


@pytest.mark.parametrize("seed", range(32))
def test_random_operator_fuzz(ctx, seed):
    """random linear operators: 1..8 terms, |alpha| <= 6 per term, d in 1..8, 0..3 coefficient
    fields, random weights, with and without the 1/sqrt(N) normalisation (Table 3 ablation)"""
    g = np.random.default_rng(1000 + seed)
    d = int(g.integers(1, 9))
    nf = int(g.integers(0, 4))
    terms = []
    for _ in range(int(g.integers(1, 9))):
        alpha = [0] * d
        for _k in range(int(g.integers(0, 7))):
            alpha[int(g.integers(0, d))] += 1
        field = int(g.integers(-1, nf)) if nf else -1
        terms.append((tuple(alpha), float(g.normal()), field))
    F, n = int(g.integers(1, 300)), int(g.integers(1, 1500))
    W = g.normal(0, g.uniform(0.5, 3), (F, d))
    b = g.uniform(0, 2 * math.pi, F)
    X = g.random((n, d))
    fields = np.ascontiguousarray(g.normal(size=(n, nf))) if nf else None
    vals = g.normal(size=n)
    weight = float(g.uniform(0.1, 50))
    normalize = bool(seed % 2)

    class B:
        pass
    h = B()
    h.X, h.terms, h.weight, h.values, h.fields = X, terms, weight, vals, fields
    dv = fls.Block(torch.from_numpy(X).cuda(), terms, weight, torch.from_numpy(vals).cuda(),
                   torch.from_numpy(fields).cuda() if nf else None)
    Ab, lda = fls.fls_assemble(ctx, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(), [dv],
                               normalize=normalize)
    fls.fls_sync(ctx)
    Ao, ro, S = oracle.assemble(W, b, [h], normalize=normalize)
    Ag, rg = rows_from_colmajor(Ab, lda, F, np.arange(n))
    emax, _ = scaled_err(Ag, Ao, S)
    assert emax <= ENTRY_TOL, (emax, d, terms)
    assert np.array_equal(rg, ro)
    # the row-major kernel holds bit-identical entries for every operator family
    Arm, rrm = fls.fls_assemble(ctx, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(), [dv],
                                normalize=normalize, layout=fls.FLS_ROW_MAJOR)
    assert np.array_equal(Arm[:, :F].cpu().numpy(), Ag) and np.array_equal(rrm.cpu().numpy(), rg)
    # A beta without materialising A (fls_eval_block) for the same operator family
    beta_h = g.normal(size=F)
    got = fls.fls_eval_block(ctx, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(),
                             torch.from_numpy(beta_h).cuda(), dv, normalize=normalize).cpu().numpy()
    assert np.abs(got - Ao @ beta_h).max() <= 1e-12 * max((S @ np.abs(beta_h)).max(), 1e-300)


@pytest.mark.parametrize("d", [1, 2, 4, 6, 8])
def test_all_dims(ctx, d):
    _mode_case(ctx, wl.op_laplacian(d, -1.0) + wl.op_identity(d, 2.0), d=d, F=150, n=300, seed=d)


# ------------------------------------------------------------------------------------- errors
def test_error_paths(ctx):
    from paper_2602_10541_b200._abi import FlsError
    p = wl.make_problem("c1_poisson1d", "mini")
    _, _, Wd, bd = _parity_feats(p)
    blocks = dev_blocks(p)
    with pytest.raises(FlsError, match="EINVAL"):
        fls.fls_assemble(ctx, Wd, bd, blocks, row_begin=0, row_end=p.n_rows + 1)
    with pytest.raises(FlsError, match="EINVAL"):
        fls.fls_assemble(ctx, Wd, bd, blocks, lda=10)
    bad = [fls.Block(blocks[0].X, [((1, 1), 1.0, -1)], 1.0, blocks[0].values)]
    with pytest.raises(FlsError, match="EINVAL"):                      # alpha beyond dim
        fls.fls_assemble(ctx, Wd, bd, bad)
    bad = [fls.Block(blocks[0].X, [((0,), 1.0, 0)], 1.0, blocks[0].values)]
    with pytest.raises(FlsError, match="EINVAL"):                      # field without fields
        fls.fls_assemble(ctx, Wd, bd, bad)
    with pytest.raises(FlsError, match="EINVAL"):
        fls.fls_features(ctx, 0, 10, 1.0, 0)
    with pytest.raises(FlsError, match="EINVAL"):
        fls.fls_features(ctx, 2, 10, -1.0, 0)
    # non-finite input is reported asynchronously at the next sync
    Xn = blocks[0].X.clone()
    Xn[5, 0] = float("nan")
    nb = [fls.Block(Xn, blocks[0].terms, 1.0, blocks[0].values)]
    fls.fls_assemble(ctx, Wd, bd, nb)
    with pytest.raises(FlsError, match="ENONFINITE"):
        fls.fls_sync(ctx)
    fls.fls_sync(ctx)                                                  # flag cleared
    # rank deficiency: a zero column without ridge
    M = torch.zeros((3 * 8,), dtype=torch.float64, device="cuda")
    M.view(3, 8)[0, :] = 1.0
    M.view(3, 8)[2, :] = 1.0
    with pytest.raises(FlsError, match="ERANK"):
        fls.fls_solve(ctx, M, 8, 8, 2)


def test_error_paths_extended(ctx):
    """argument errors of the non-assembly entry points return FLS_EINVAL / FLS_EUNSUPPORTED"""
    from paper_2602_10541_b200._abi import FlsError
    dev = "cuda"
    with pytest.raises(FlsError, match="EINVAL"):
        fls.fls_sample_box(ctx, 2, 10, [0, 1], [1, 1], seed=0)          # lo == hi on axis 1
    with pytest.raises(FlsError, match="EINVAL"):
        fls.fls_features_blocks(ctx, 2, [10, 0], [1.0, 2.0], 0)         # empty block
    with pytest.raises(FlsError, match="EINVAL"):
        fls.fls_features_blocks(ctx, 2, [10], [-1.0], 0)
    A = torch.randn(10 * 3, dtype=torch.float64, device=dev)
    with pytest.raises(FlsError, match="EINVAL"):
        fls.QRFactor(ctx, A, 2, 10, 3)                                   # 2 rows < 3 features
    u = torch.zeros(5, dtype=torch.float64, device=dev)
    bad = fls.make_nonlinearity("poly", [0.0] * 3)
    bad.degree = 9
    with pytest.raises(FlsError, match="EINVAL"):
        fls.fls_nl_residual(ctx, bad, u, u, u)
    X = torch.rand((20, 2), dtype=torch.float64, device=dev)
    W = torch.randn((7, 2), dtype=torch.float64, device=dev)
    b = torch.rand(7, dtype=torch.float64, device=dev)
    blk = fls.Block(X, [((0, 0), 1.0, 0)], 1.0, torch.zeros(20, dtype=torch.float64, device=dev),
                    torch.ones((20, 1), dtype=torch.float64, device=dev))
    G = fls.fls_bandwidth_grad(ctx, W, W, b, [blk], torch.zeros(7, dtype=torch.float64, device=dev))
    assert np.all(np.array(G) == 0.0)                                    # r = 0: fields allowed
    blk_bad = fls.Block(X, [((0, 0), 1.0, 1)], 1.0, torch.zeros(20, dtype=torch.float64, device=dev),
                        torch.ones((20, 1), dtype=torch.float64, device=dev))
    with pytest.raises(FlsError, match="EINVAL"):                        # field id >= n_fields
        fls.fls_bandwidth_grad(ctx, W, W, b, [blk_bad], torch.zeros(7, dtype=torch.float64, device=dev))
    with pytest.raises(FlsError, match="EINVAL"):                        # eval op with a field
        fls.fls_eval(ctx, W, b, torch.zeros(7, dtype=torch.float64, device=dev), X,
                     terms=[((0, 0), 1.0, 0)])
    fls.fls_sync(ctx)
    # FLS_ENOMEM: a workspace request far beyond the device (10^10 features), raw ABI call
    import ctypes as C
    from paper_2602_10541_b200 import _abi
    bs = fls.BlockSet([fls.Block(X, [((2, 0), 1.0, -1)], 1.0, None)], 2)
    A = torch.empty(64, dtype=torch.float64, device=dev)
    st = _abi.load().fls_assemble(ctx.handle, C.c_void_p(W.data_ptr()), C.c_void_p(b.data_ptr()), 2,
                                  10 ** 10, 1, bs.arr, 1, 0, 20, C.c_void_p(A.data_ptr()), 20, 0, None)
    assert _abi.STATUS[st] == "FLS_ENOMEM", _abi.load().fls_last_error()


# ------------------------------------------------------------------------------------- solve + eval
@pytest.mark.parametrize("name,size", [("c1_poisson1d", "full"), ("c2_poisson2d", "full"),
                                       ("c3_poisson5d", "mini"), ("c4_heat2d", "mini"),
                                       ("c5_biharm3d", "mini")])
def test_solve_and_eval_parity(ctx, name, size):
    p = wl.make_problem(name, size)
    W, b, Wd, bd = _parity_feats(p)
    F, R = p.n_features, p.n_rows
    ridge = p.ridge_rel > 0
    Ab, lda = fls.fls_assemble(ctx, Wd, bd, dev_blocks(p), extra_rows=F if ridge else 0)
    if ridge:   # the relative ridge computed inside libfls == the absolute one from fls_frob2
        Ab2 = Ab.clone()
        sq = p.ridge_rel * math.sqrt(fls.fls_frob2(ctx, Ab2, R, lda, F))
        beta2, res2 = fls.fls_solve_mu(ctx, Ab2, R, lda, F, sq)
    beta, res = fls.fls_solve(ctx, Ab, R, lda, F, p.ridge_rel)   # sqrt(mu) = tau ||A||_F inside
    if ridge:
        assert torch.equal(beta, beta2) and res == res2
    Xt = p.test_points(10_000)
    u_gpu = fls.fls_eval(ctx, Wd, bd, beta, torch.from_numpy(Xt).cuda()).cpu().numpy()
    # oracle chain
    Ao, ro, _ = oracle.assemble(W, b, p.blocks, want_scale=False)
    beta_o, res_o, _ = oracle.lstsq(Ao, ro, ridge_rel=p.ridge_rel)
    u_orc = oracle.evaluate(W, b, beta_o, Xt)
    rel = np.linalg.norm(u_gpu - u_orc) / np.linalg.norm(u_orc)
    assert rel <= U_TOL, rel
    # eval parity alone (same beta on both sides)
    u_gpu2 = fls.fls_eval(ctx, Wd, bd, torch.from_numpy(beta_o).cuda(),
                          torch.from_numpy(Xt).cuda()).cpu().numpy()
    scale = np.abs(beta_o).sum() / math.sqrt(F)
    assert np.abs(u_gpu2 - u_orc).max() <= 1e-12 * max(scale, 1.0)


def test_eval_with_operator_matches_assembled_rows(ctx):
    p = wl.make_problem("c4_heat2d", "mini")
    W, b, Wd, bd = _parity_feats(p)
    F = p.n_features
    beta = torch.from_numpy(np.random.default_rng(0).normal(size=F)).cuda()
    X = torch.from_numpy(p.test_points(999)).cuda()
    terms = p.blocks[0].terms
    Lu = fls.fls_eval(ctx, Wd, bd, beta, X, terms=terms).cpu().numpy()

    class B:
        pass
    h = B()
    h.X, h.terms, h.weight, h.values, h.fields = X.cpu().numpy(), terms, 1.0, None, None
    Ao, _, S = oracle.assemble(W, b, [h])
    ref = Ao @ beta.cpu().numpy()
    assert np.abs(Lu - ref).max() <= 1e-12 * (S @ np.abs(beta.cpu().numpy())).max()


@pytest.mark.parametrize("name", ["c5_biharm3d", "c4_heat2d", "c2_poisson2d"])
def test_eval_block_matches_oracle_rows(ctx, name):
    """fls_eval_block = A_block beta with the block's weight and coefficient fields (C5: the
    16 (1 + x1) u term), A never materialised; every block of the problem"""
    p = wl.make_problem(name, "mini")
    W, b, Wd, bd = _parity_feats(p)
    F = p.n_features
    beta_h = np.random.default_rng(1).normal(size=F)
    beta = torch.from_numpy(beta_h).cuda()
    for blk, dblk in zip(p.blocks, dev_blocks(p)):
        got = fls.fls_eval_block(ctx, Wd, bd, beta, dblk).cpu().numpy()
        Ao, _, S = oracle.assemble(W, b, [blk])
        ref = Ao @ beta_h
        assert np.abs(got - ref).max() <= 1e-12 * (S @ np.abs(beta_h)).max(), blk.name


def test_eval_block_two_fields_mixed_parity(ctx):
    """mixed-parity operator with two coefficient fields (the sin+cos eval path)"""
    rng = np.random.default_rng(5)
    d, F, n = 3, 211, 777
    W = rng.normal(0, 2.0, size=(F, d))
    b = rng.uniform(0, 2 * np.pi, size=F)
    X = rng.uniform(0, 1, size=(n, d))
    fields = rng.normal(size=(n, 3))
    terms = [((2, 0, 0), 1.0, -1), ((0, 1, 0), -0.5, 2), ((0, 0, 0), 3.0, 0), ((1, 1, 1), 0.25, 2)]

    class B:
        pass
    h = B()
    h.X, h.terms, h.weight, h.values, h.fields = X, terms, 7.0, None, fields
    Ao, _, S = oracle.assemble(W, b, [h])
    beta_h = rng.normal(size=F)
    blk = fls.Block(torch.from_numpy(X).cuda(), terms, 7.0, None, torch.from_numpy(fields).cuda())
    got = fls.fls_eval_block(ctx, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(),
                             torch.from_numpy(beta_h).cuda(), blk).cpu().numpy()
    assert np.abs(got - Ao @ beta_h).max() <= 1e-12 * (S @ np.abs(beta_h)).max()
    bad = fls.Block(torch.from_numpy(X).cuda(), [((0, 0, 0), 1.0, 5)], 1.0, None,
                    torch.from_numpy(fields).cuda())
    with pytest.raises(fls.FlsError):
        fls.fls_eval_block(ctx, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(),
                           torch.from_numpy(beta_h).cuda(), bad)


# ------------------------------------------------------------------------------------- host path
@pytest.mark.parametrize("chunk", [0, 1000, 4096])
def test_assemble_host_matches_device(ctx, chunk):
    """fls_assemble_host (host buffers, chunked, two streams) == fls_assemble, bitwise."""
    p = wl.make_problem("c4_heat2d", "mini")
    W, b, Wd, bd = _parity_feats(p)
    F, R = p.n_features, p.n_rows
    Ab, lda = fls.fls_assemble(ctx, Wd, bd, dev_blocks(p))
    ref = Ab[: (F + 1) * lda].view(F + 1, lda)[:, :R].cpu().numpy()
    for (r0, r1) in [(0, R), (17, R - 5)]:
        n = r1 - r0
        ldh = n + 3
        A_h = np.full((F + 1) * ldh, np.nan)
        fls.fls_assemble_host(ctx, W, b, p.blocks, A_h, ldh, A_h[F * ldh:], row_begin=r0,
                              row_end=r1, chunk_rows=chunk)
        got = A_h.reshape(F + 1, ldh)[:, :n]
        assert np.array_equal(got, ref[:, r0:r1])
        assert np.isnan(A_h.reshape(F + 1, ldh)[:F, n:]).all()     # padding untouched


# ------------------------------------------------------------------------------------- TSQR on one GPU
@pytest.mark.parametrize("name,size,P", [("c1_poisson1d", "full", 8), ("c2_poisson2d", "full", 4),
                                         ("c5_biharm3d", "mini", 3)])
def test_tsqr_logical_blocks_match_oracle(ctx, name, size, P):
    """TSQR (per-block fls_qr_r, stacked R factors, root fls_solve) over P row shards held on
    one device; C1 at P=8 has 125-row blocks < F+1 (trapezoidal R).  u vs oracle lstsq."""
    from paper_2602_10541_b200.dist import tsqr_local
    p = wl.make_problem(name, size)
    W, b, Wd, bd = _parity_feats(p)
    F, R = p.n_features, p.n_rows
    bset = fls.BlockSet(dev_blocks(p), p.dim)
    blocks = []
    for r in range(P):
        a, e = wl.shard_range(R, r, P)
        Ab, lda = fls.fls_assemble(ctx, Wd, bd, bset, row_begin=a, row_end=e)
        blocks.append((Ab, e - a, lda))
    beta, _ = tsqr_local(blocks, F, ridge_rel=p.ridge_rel, ctx=ctx)
    Xt = p.test_points(10_000)
    u_gpu = fls.fls_eval(ctx, Wd, bd, beta, torch.from_numpy(Xt).cuda()).cpu().numpy()
    Ao, ro, _ = oracle.assemble(W, b, p.blocks, want_scale=False)
    beta_o, _, _ = oracle.lstsq(Ao, ro, ridge_rel=p.ridge_rel)
    u_orc = oracle.evaluate(W, b, beta_o, Xt)
    assert np.linalg.norm(u_gpu - u_orc) / np.linalg.norm(u_orc) <= U_TOL


# ------------------------------------------------------------------------------------- full-size solves
@pytest.mark.parametrize("name", ["c3_poisson5d", "c4_heat2d", "c5_biharm3d"])
def test_full_size_solve_parity_with_oracle_artifact(ctx, name):
    """Fitted u at the 10,000 held-out points at BASELINE size (C5: its 262,144-row solve subset)
    vs tests/golden/oracle_u_<cfg>.npz, written offline by tools/make_oracle_artifacts.py from
    oracle/ only (Householder QR of the oracle's own term-by-term assembly)."""
    import os
    art = os.path.join(os.path.dirname(__file__), "golden", f"oracle_u_{name}.npz")
    if not os.path.exists(art):
        pytest.skip(f"no oracle artifact {art}")
    u_orc = np.load(art)["u_test"]
    kw = {"n_int": 262_144} if name == "c5_biharm3d" else {}
    p = wl.make_problem(name, "full", **kw)
    W, b, Wd, bd = _parity_feats(p)
    F, R = p.n_features, p.n_rows
    ridge = p.ridge_rel > 0
    Ab, lda = fls.fls_assemble(ctx, Wd, bd, dev_blocks(p), extra_rows=F if ridge else 0)
    beta, _ = fls.fls_solve(ctx, Ab, R, lda, F, p.ridge_rel)
    del Ab
    torch.cuda.empty_cache()
    Xt = p.test_points(10_000)
    u_gpu = fls.fls_eval(ctx, Wd, bd, beta, torch.from_numpy(Xt).cuda()).cpu().numpy()
    rel = np.linalg.norm(u_gpu - u_orc) / np.linalg.norm(u_orc)
    assert rel <= U_TOL, rel


# ------------------------------------------------------------------------------------- Alg. 1 line 2 + pipeline
def test_sample_points_match_oracle(ctx):
    lo, hi = [0.0, -1.0, 2.0], [1.0, 1.0, 2.5]
    Xd = fls.fls_sample_box(ctx, 3, 1001, lo, hi, seed=7, stream=3).cpu().numpy()
    Xo = oracle.sample_box(3, 1001, lo, hi, 7, 3)
    assert np.array_equal(Xd, Xo)
    Fd = fls.fls_sample_faces(ctx, 3, 37, [0, 2], lo, hi, seed=7, stream=4).cpu().numpy()
    Fo = oracle.sample_faces(3, 37, 0b101, lo, hi, 7, 4)
    assert np.array_equal(Fd, Fo)
    assert np.all(Fd[:37, 0] == 0.0) and np.all(Fd[37:74, 0] == 1.0) and np.all(Fd[111:, 2] == 2.5)


def test_pipeline_solve_linear_matches_oracle(ctx):
    """Algorithm 1 through paper_2602_10541_b200.pipeline (features on the device, points from
    fls_sample_*, operators from paper_2602_10541_b200.operators) vs the oracle chain on the
    same W, b, points."""
    from paper_2602_10541_b200 import operators as ops
    from paper_2602_10541_b200.pipeline import solve_linear
    pi = math.pi
    Xi = fls.fls_sample_box(ctx, 2, 3000, [0, 0], [1, 1], seed=0, stream=3)
    Xb = fls.fls_sample_faces(ctx, 2, 150, [0, 1], [0, 0], [1, 1], seed=0, stream=4)

    def u(X):
        return torch.sin(pi * X[:, 0]) * torch.sin(2 * pi * X[:, 1])
    f = 5 * pi * pi * u(Xi)                                  # -Lap u
    blocks = [fls.Block(Xi, ops.laplacian(2, -1.0), 1.0, f.contiguous()),
              fls.Block(Xb, ops.identity(2), 100.0, u(Xb).contiguous())]
    sol = solve_linear(ctx, dim=2, n_features=800, sigma=4.0, seed=0, blocks=blocks)
    Xt = fls.fls_sample_box(ctx, 2, 2000, [0, 0], [1, 1], seed=0, stream=6)
    ug = sol.evaluate(Xt).cpu().numpy()

    class B:
        def __init__(s, X, terms, w, v):
            s.X, s.terms, s.weight, s.values, s.fields = X, terms, w, v, None
    hb = [B(blk.X.cpu().numpy(), blk.terms, blk.weight, blk.values.cpu().numpy()) for blk in blocks]
    W, b = sol.W.cpu().numpy(), sol.b.cpu().numpy()
    Ao, ro, _ = oracle.assemble(W, b, hb, want_scale=False)
    bo, _, _ = oracle.lstsq(Ao, ro)
    uo = oracle.evaluate(W, b, bo, Xt.cpu().numpy())
    assert np.linalg.norm(ug - uo) / np.linalg.norm(uo) <= U_TOL
    us = u(Xt).cpu().numpy()
    assert np.linalg.norm(ug - us) / np.linalg.norm(us) < 1e-6
    # residual check L[u_N] vs f at the test points
    Lu = sol.evaluate(Xt, terms=ops.laplacian(2, -1.0)).cpu().numpy()
    assert np.linalg.norm(Lu - 5 * pi * pi * us) / np.linalg.norm(5 * pi * pi * us) < 1e-4


# ------------------------------------------------------------------------------------- f3 / f4
def test_features_blocks_match_oracle(ctx):
    counts, sig = [500, 7, 993], [1.0, 3.0, 12.0]
    Wd, bd = fls.fls_features_blocks(ctx, 2, counts, sig, 11)
    Wo, bo = oracle.features_blocks(2, counts, sig, 11)
    assert np.array_equal(bd.cpu().numpy(), bo)
    ulp = np.spacing(np.abs(Wo))
    assert np.all(np.abs(Wd.cpu().numpy() - Wo) <= 8 * ulp)
    W1, b1 = fls.fls_features(ctx, 2, 1500, 2.5, 11)
    Wb, bb = fls.fls_features_blocks(ctx, 2, [1500], [2.5], 11)
    assert torch.equal(W1, Wb) and torch.equal(b1, bb)


def _alt_rhs(p):
    """rhs [f; lam g; ...] of a second manufactured solution u2 on the same points (closed forms)"""
    pi = math.pi
    out = []
    for blk in p.blocks:
        X = blk.X
        if p.name == "c2_poisson2d":          # u2 = cos(pi x) y^2 + x, -Lap u2 = pi^2 cos(pi x) y^2 - 2 cos(pi x)
            u2 = np.cos(pi * X[:, 0]) * X[:, 1] ** 2 + X[:, 0]
            f2 = pi ** 2 * np.cos(pi * X[:, 0]) * X[:, 1] ** 2 - 2 * np.cos(pi * X[:, 0])
        elif p.name == "c4_heat2d":           # u2 = e^{-2t} sin(2 pi x) sin(pi y)
            u2 = np.exp(-2 * X[:, 2]) * np.sin(2 * pi * X[:, 0]) * np.sin(pi * X[:, 1])
            f2 = (-2 + 0.1 * 5 * pi ** 2) * u2
        else:                                 # c5: u2 = sin(2 pi x) sin(pi y) sin(pi z)
            u2 = np.sin(2 * pi * X[:, 0]) * np.sin(pi * X[:, 1]) * np.sin(pi * X[:, 2])
            f2 = (36 * pi ** 4 + 16 * (1 + X[:, 0])) * u2
        out.append(blk.weight * (f2 if blk.name == "pde" else u2))
    return np.concatenate(out)


@pytest.mark.parametrize("name,size", [("c2_poisson2d", "full"), ("c4_heat2d", "mini"),
                                       ("c5_biharm3d", "mini")])
def test_cached_qr_many_rhs(ctx, name, size):
    """App. I matrix caching: factor A once, solve several right-hand sides;
    each fitted u matches the oracle's full lstsq of [A | b_k] within 1e-6."""
    p = wl.make_problem(name, size)
    W, b, Wd, bd = _parity_feats(p)
    F, R = p.n_features, p.n_rows
    Ab, lda = fls.fls_assemble(ctx, Wd, bd, dev_blocks(p))
    sq = p.ridge_rel * math.sqrt(fls.fls_frob2(ctx, Ab, R, lda, F)) if p.ridge_rel > 0 else 0.0
    qr = fls.QRFactor(ctx, Ab, R, lda, F, sq)
    rhs0 = Ab[F * lda: F * lda + R].cpu().numpy()
    rhs1 = _alt_rhs(p)
    # well-posed right-hand sides only (manufactured solutions): with a numerically rank-deficient
    # A the fitted u of an arbitrary rhs is not unique across QR variants
    B = np.stack([rhs0, rhs1, 2.0 * rhs0 - 0.5 * rhs1], axis=1)                         # (R, 3)
    Bd = torch.from_numpy(np.ascontiguousarray(B.T)).cuda().reshape(-1)                 # col-major
    Beta = qr.solve(Bd, ldb=R)
    Xt = p.test_points(10_000)
    Xd = torch.from_numpy(Xt).cuda()
    Ao, _, _ = oracle.assemble(W, b, p.blocks, want_scale=False)
    for k in range(3):
        u_gpu = fls.fls_eval(ctx, Wd, bd, Beta[k].contiguous(), Xd).cpu().numpy()
        beta_o, _, _ = oracle.lstsq(Ao, B[:, k], ridge_rel=p.ridge_rel)
        u_orc = oracle.evaluate(W, b, beta_o, Xt)
        rel = np.linalg.norm(u_gpu - u_orc) / np.linalg.norm(u_orc)
        assert rel <= U_TOL, (k, rel)
    qr.close()


# ------------------------------------------------------------------------------------- fused a1+a2
@pytest.mark.parametrize("fuse", ["0", "1000000000000"])
@pytest.mark.parametrize("name", ["c1_poisson1d", "c2_poisson2d", "c3_poisson5d", "c4_heat2d",
                                  "c5_biharm3d"])
def test_features_assemble_fused_bit_identical(ctx, name, fuse, monkeypatch):
    """fls_features_assemble == fls_features then fls_assemble, bit for bit: one block batch
    (fused prefactors), more blocks than one prefactor batch holds, shards and row-major.
    fuse = FLS_FUSE_MAX_ENTRIES: "0" = two launches (features + prefactors, then assembly),
    1e12 = ONE launch whose CTAs draw and fold their own features' records (the default for
    calls up to 2^25 entries: C1, C2)"""
    monkeypatch.setenv("FLS_FUSE_MAX_ENTRIES", fuse)
    p = wl.make_problem(name, "mini")
    F, d = p.n_features, p.dim
    sigma, seed = float(p.sigma), int(p.seed)
    Wd, bd = fls.fls_features(ctx, d, F, sigma, seed)
    base = dev_blocks(p)
    for blks in (base, base + base):
        bs = fls.BlockSet(blks, d)
        ref, lda = fls.fls_assemble(ctx, Wd, bd, bs)
        W2, b2, got, lda2 = fls.fls_features_assemble(ctx, d, F, sigma, seed, bs)
        fls.fls_sync(ctx)
        assert lda2 == lda
        assert torch.equal(W2, Wd) and torch.equal(b2, bd)
        R = bs.total

        def cols(Ab, ld, n):   # (F + 1, n) valid part of a flat column-major [A | b]
            return Ab[: (F + 1) * ld].view(F + 1, ld)[:, :n]
        nbad = int((cols(got, lda, R) != cols(ref, lda, R)).sum())
        assert nbad == 0, (len(blks), nbad)
        a, e = wl.shard_range(R, 1, 3)
        ref_s, ls = fls.fls_assemble(ctx, Wd, bd, bs, row_begin=a, row_end=e)
        _, _, got_s, _ = fls.fls_features_assemble(ctx, d, F, sigma, seed, bs, row_begin=a,
                                                   row_end=e)
        Arm, rrm = fls.fls_assemble(ctx, Wd, bd, bs, layout=fls.FLS_ROW_MAJOR)
        _, _, Arm2, rrm2 = fls.fls_features_assemble(ctx, d, F, sigma, seed, bs,
                                                     layout=fls.FLS_ROW_MAJOR)
        fls.fls_sync(ctx)
        assert torch.equal(cols(got_s, ls, e - a), cols(ref_s, ls, e - a))
        assert torch.equal(Arm2[:, :F], Arm[:, :F]) and torch.equal(rrm2, rrm)
    with pytest.raises(fls.FlsError):
        fls.fls_features_assemble(ctx, d, F, -1.0, seed, base)


@pytest.mark.parametrize("fuse", ["0", "1000000000000"])
@pytest.mark.parametrize("name,size", [("c1_poisson1d", "full"), ("c2_poisson2d", "full"),
                                       ("c4_heat2d", "mini")])
def test_batch_plan_does_not_change_entries(ctx, name, size, fuse, monkeypatch):
    """the joint launch plan of a multi-block batch (FLS_BATCH_PLAN 0-3: per-block grids, capped
    features per CTA, one feature count, equal entries) only moves work between CTAs: [A | b]
    is bit-identical for every strategy, fused and unfused, and matches the oracle"""
    monkeypatch.setenv("FLS_FUSE_MAX_ENTRIES", fuse)
    p = wl.make_problem(name, size)
    F, d = p.n_features, p.dim
    bs = fls.BlockSet(dev_blocks(p), d)
    R = bs.total
    outs = []
    for plan in ("0", "1", "2", "3"):
        monkeypatch.setenv("FLS_BATCH_PLAN", plan)
        Wd, bd, Ab, lda = fls.fls_features_assemble(ctx, d, F, float(p.sigma), int(p.seed), bs)
        fls.fls_sync(ctx)
        outs.append(Ab[: (F + 1) * lda].view(F + 1, lda)[:, :R].clone())
    for k in range(1, 4):
        assert torch.equal(outs[k], outs[0]), k
    W, b = Wd.cpu().numpy(), bd.cpu().numpy()   # the entries' parity for the drawn features
    rows = np.unique(np.linspace(0, R - 1, 64).astype(np.int64))
    Ao, ro, S = oracle.assemble(W, b, p.blocks, rows=rows)
    M = outs[0].cpu().numpy()
    emax, _ = scaled_err(M[:F, rows].T, Ao, S)
    assert emax <= ENTRY_TOL, emax
    assert np.array_equal(M[F, rows], ro)


@pytest.mark.parametrize("fuse", ["0", "1000000000000"])
@pytest.mark.parametrize("name,size", [("c1_poisson1d", "full"), ("c2_poisson2d", "full"),
                                       ("c3_poisson5d", "mini"), ("c4_heat2d", "mini")])
def test_guided_tail_does_not_change_entries(ctx, name, size, fuse, monkeypatch):
    """the launch plan's guided tail (each block's last FLS_TAIL_PCT % of features in narrower
    CTAs dispatched after every main CTA; default on for unfused launches of 2^22..2^25
    entries) only moves work between CTAs: [A | b] and W, b are bit-identical with and without
    it, fused and unfused, for tails that split feature chunks unevenly (odd per-CTA counts,
    a tail narrower than one CTA), and the entries match the oracle"""
    monkeypatch.setenv("FLS_FUSE_MAX_ENTRIES", fuse)
    p = wl.make_problem(name, size)
    F, d = p.n_features, p.dim
    bs = fls.BlockSet(dev_blocks(p), d)
    R = bs.total
    outs = []
    for pct, fpc in (("0", "4"), ("10", "4"), ("5", "3"), ("33", "2"), ("50", "1000")):
        monkeypatch.setenv("FLS_TAIL_PCT", pct)
        monkeypatch.setenv("FLS_TAIL_FPC", fpc)
        Wd, bd, Ab, lda = fls.fls_features_assemble(ctx, d, F, float(p.sigma), int(p.seed), bs)
        fls.fls_sync(ctx)
        outs.append((Ab[: (F + 1) * lda].view(F + 1, lda)[:, :R].clone(), Wd.clone(), bd.clone()))
    for k in range(1, len(outs)):
        for t in range(3):
            assert torch.equal(outs[k][t], outs[0][t]), (k, t)
    W, b = outs[0][1].cpu().numpy(), outs[0][2].cpu().numpy()
    rows = np.unique(np.linspace(0, R - 1, 64).astype(np.int64))
    Ao, ro, S = oracle.assemble(W, b, p.blocks, rows=rows)
    M = outs[0][0].cpu().numpy()
    emax, _ = scaled_err(M[:F, rows].T, Ao, S)
    assert emax <= ENTRY_TOL, emax
    assert np.array_equal(M[F, rows], ro)


def test_guided_tail_keeps_the_phase_guard(ctx, monkeypatch):
    """a phase out of range inside a tail segment's features still raises FLS_EUNSUPPORTED"""
    monkeypatch.setenv("FLS_TAIL_PCT", "25")
    monkeypatch.setenv("FLS_TAIL_FPC", "2")
    p = wl.make_problem("c2_poisson2d", "mini")
    F, d = p.n_features, p.dim
    W, b = p.parity_features()
    W = W.copy()
    W[F - 1, :] = 5e4          # the last feature sits in the tail: |W.x| > FLS_MAX_PHASE
    bs = fls.BlockSet(dev_blocks(p), d)
    from paper_2602_10541_b200._abi import FlsError
    fls.fls_assemble(ctx, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(), bs)
    with pytest.raises(FlsError, match="EUNSUPPORTED"):
        fls.fls_sync(ctx)
    fls.fls_sync(ctx)                                        # flag cleared


def test_pdl_off_gives_identical_entries(ctx, tmp_path):
    """FLS_PDL=0 (assembly launched without programmatic dependent launch, read once per
    process) writes the same bits as the default PDL launch, for the fused and unfused calls"""
    import subprocess
    import sys
    script = tmp_path / "asm.py"
    script.write_text(
        "import sys, torch\n"
        f"sys.path.insert(0, {str(wl.__file__.rsplit('/workloads/', 1)[0])!r})\n"
        "sys.path.insert(0, sys.argv[2])\n"
        "import workloads as wl\n"
        "from gpu_common import dev_blocks\n"
        "from paper_2602_10541_b200 import fls\n"
        "p = wl.make_problem('c3_poisson5d', 'mini')\n"
        "ctx = fls.Context()\n"
        "bs = fls.BlockSet(dev_blocks(p), p.dim)\n"
        "W, b, A, lda = fls.fls_features_assemble(ctx, p.dim, p.n_features, p.sigma, p.seed, bs)\n"
        "A2, _ = fls.fls_assemble(ctx, W, b, bs)\n"
        "fls.fls_sync(ctx)\n"
        "torch.save({'A': A.cpu(), 'A2': A2.cpu(), 'lda': lda}, sys.argv[1])\n")
    import os
    here = os.path.dirname(os.path.abspath(__file__))
    outs = []
    for pdl in ("1", "0"):
        out = tmp_path / f"a{pdl}.pt"
        env = dict(os.environ, FLS_PDL=pdl)
        r = subprocess.run([sys.executable, str(script), str(out), here], env=env,
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(torch.load(out))
    p = wl.make_problem("c3_poisson5d", "mini")
    F, R, lda = p.n_features, p.n_rows, outs[0]["lda"]
    for key in ("A", "A2"):
        a, b = (o[key][: (F + 1) * lda].view(F + 1, lda)[:, :R] for o in outs)
        assert torch.equal(a, b), key


def test_binding_rejects_wrong_shapes_and_small_buffers(ctx):
    """the thin binding validates what the C ABI cannot see (tensor sizes, shapes, devices)
    before the call: a wrong shape or a short buffer would otherwise be written out of bounds"""
    p = wl.make_problem("c1_poisson1d", "mini")
    _, _, Wd, bd = _parity_feats(p)
    blocks = dev_blocks(p)
    F, R = p.n_features, p.n_rows
    with pytest.raises(ValueError, match="X must be"):
        fls.fls_assemble(ctx, Wd, bd, [fls.Block(blocks[0].X.view(-1, 1).repeat(1, 2), blocks[0].terms)])
    with pytest.raises(ValueError, match="values has"):
        fls.fls_assemble(ctx, Wd, bd, [fls.Block(blocks[0].X, blocks[0].terms, 1.0, blocks[0].values[:-1])])
    with pytest.raises(ValueError, match="fields must be"):
        fls.fls_assemble(ctx, Wd, bd, [fls.Block(blocks[0].X, blocks[0].terms, 1.0, None,
                                                 torch.ones((3, 1), dtype=torch.float64, device="cuda"))])
    with pytest.raises(ValueError, match="b has"):
        fls.fls_assemble(ctx, Wd, bd[:-1], blocks)
    lda = fls.round_up(R, 4)
    short = torch.empty((F * lda,), dtype=torch.float64, device="cuda")      # no room for column F
    with pytest.raises(ValueError, match="rhs holds"):
        fls.fls_assemble(ctx, Wd, bd, blocks, A=short, lda=lda)
    with pytest.raises(ValueError, match="A holds"):
        fls.fls_assemble(ctx, Wd, bd, blocks, A=short[: (F - 1) * lda], lda=lda, with_rhs=False)
    with pytest.raises(ValueError, match="beta holds"):
        fls.fls_eval(ctx, Wd, bd, torch.zeros(F - 1, dtype=torch.float64, device="cuda"), blocks[0].X)
    with pytest.raises(ValueError, match="Ab holds"):
        fls.fls_solve(ctx, short[:100], R, lda, F)


# ------------------------------------------------------------------------- phase-range guard
def _guard_case(zmax_target, d=1, n=3000, F=300, seed=0):
    """features with |W_j| ~ zmax_target on x in [0.5, 1]^d: max |z| ~ zmax_target"""
    g = np.random.default_rng(seed)
    W = g.uniform(0.5, 1.0, (F, d)) * (zmax_target / d) * np.where(g.random((F, d)) < 0.5, -1, 1)
    b = g.uniform(0, 2 * np.pi, F)
    X = g.uniform(0.5, 1.0, (n, d))
    z = X @ W.T + b
    return W, b, X, float(np.abs(z).max())


@pytest.mark.parametrize("layout", ["col", "row"])
def test_phase_beyond_limit_reports_unsupported(ctx, layout):
    """|z| > FLS_MAX_PHASE = 1e4 -> FLS_EUNSUPPORTED at the next fls_sync (no silent garbage);
    just below the limit -> no error, entries within the documented error at that |z|"""
    from paper_2602_10541_b200._abi import FlsError
    lay = fls.FLS_COL_MAJOR if layout == "col" else fls.FLS_ROW_MAJOR
    W, b, X, zmax = _guard_case(3.0e4)
    assert zmax > 1e4
    blk = [fls.Block(torch.from_numpy(X).cuda(), [((2,), -1.0, -1)], 1.0)]
    fls.fls_assemble(ctx, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(), blk, layout=lay)
    with pytest.raises(FlsError, match="EUNSUPPORTED"):
        fls.fls_sync(ctx)
    fls.fls_sync(ctx)                                        # flag cleared
    W, b, X, zmax = _guard_case(9.0e3)
    assert 5e3 < zmax < 1e4
    blk = [fls.Block(torch.from_numpy(X).cuda(), [((2,), -1.0, -1)], 1.0)]
    A, _ = fls.fls_assemble(ctx, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(), blk, layout=lay)
    fls.fls_sync(ctx)
    F, n = W.shape[0], X.shape[0]
    M = (A[: F * fls.round_up(n, 4)].view(F, -1)[:, :n].T if layout == "col"
         else A.view(n, -1)[:, :F]).cpu().numpy()
    class _OBlk:
        pass
    h = _OBlk()
    h.X, h.terms, h.weight, h.values, h.fields = X, [((2,), -1.0, -1)], 1.0, np.zeros(n), None
    Ao, _, S = oracle.assemble(W, b, [h])
    err = (np.abs(M - Ao) / S).max()
    # rounding of z itself: ~ a few ulp(|z|) ~ 1e-12 x |z| / 1e4 relative to S
    assert err <= 8 * np.spacing(zmax), err


def test_phase_bound_exceeded_but_phase_in_range_is_not_an_error(ctx):
    """the per-CTA bound ||W_j||_1 ||x_i||_inf + |b_j| can exceed the limit while every actual
    |z| is small: the exact re-check keeps such inputs valid (no false positive)"""
    g = np.random.default_rng(1)
    F, n = 256, 2048
    W = np.zeros((F, 2))
    W[:, 0] = g.uniform(5e5, 1e6, F)                         # ||W_j||_1 ~ 1e6
    b = g.uniform(0, 2 * np.pi, F)
    X = np.stack([g.uniform(0, 1e-3, n), g.uniform(10, 50, n)], 1)   # ||x||_inf ~ 50, z = W0 x0 + b <= 1e3
    z = X @ W.T + b
    assert np.abs(z).max() < 1.01e3
    blk = [fls.Block(torch.from_numpy(X).cuda(), [((0, 0), 1.0, -1)], 1.0)]
    Wd, bd = torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda()
    for lay in (fls.FLS_COL_MAJOR, fls.FLS_ROW_MAJOR):
        fls.fls_assemble(ctx, Wd, bd, blk, layout=lay)
        fls.fls_sync(ctx)                                    # no FLS_EUNSUPPORTED
    u = fls.fls_eval(ctx, Wd, bd, torch.ones(F, dtype=torch.float64, device="cuda"),
                     torch.from_numpy(X).cuda())
    fls.fls_sync(ctx)
    assert np.allclose(u.cpu().numpy(), np.sin(z).sum(1) / np.sqrt(F), rtol=0, atol=1e-10)


def test_eval_phase_beyond_limit_reports_unsupported(ctx):
    from paper_2602_10541_b200._abi import FlsError
    W, b, X, zmax = _guard_case(2.0e4, d=2)
    u = fls.fls_eval(ctx, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(),
                     torch.ones(W.shape[0], dtype=torch.float64, device="cuda"), torch.from_numpy(X).cuda())
    with pytest.raises(FlsError, match="EUNSUPPORTED"):
        fls.fls_sync(ctx)


def test_back_to_back_calls_with_pdl_overlap_keep_stream_order(ctx):
    """the feature / prefactor kernel of call k+1 starts (programmatic dependent launch) while
    call k's assembly still runs, and call k+1's assembly launches early too: every write of
    call k+1 must still land after call k's.  Alternate two sets of rhs values (and two seeds)
    into the SAME [A | b] many times; the buffer must always hold the last call's result."""
    p = wl.make_problem("c2_poisson2d", "full")
    d, F, R = p.dim, p.n_features, p.n_rows
    base = dev_blocks(p)
    alt = [fls.Block(b.X, b.terms, b.weight, -3.0 * b.values + 1.0, b.fields) for b in base]
    sets = [fls.BlockSet(base, d), fls.BlockSet(alt, d)]
    lda = fls.round_up(R, 4)
    refs = []
    for k in range(2):
        W, b, A, _ = fls.fls_features_assemble(ctx, d, F, p.sigma, k, sets[k], lda=lda)
        fls.fls_sync(ctx)
        refs.append((W.clone(), b.clone(), A[: (F + 1) * lda].clone()))
    A = torch.empty(((F + 1) * lda,), dtype=torch.float64, device="cuda")
    W = torch.empty((F, d), dtype=torch.float64, device="cuda")
    b = torch.empty((F,), dtype=torch.float64, device="cuda")
    for n in (1, 2, 3, 8, 15):
        for i in range(n):
            fls.fls_features_assemble(ctx, d, F, p.sigma, i % 2, sets[i % 2], W=W, b=b, A=A, lda=lda)
        fls.fls_sync(ctx)
        last = (n - 1) % 2
        assert torch.equal(W, refs[last][0]) and torch.equal(b, refs[last][1])
        V, Vr = A.view(F + 1, lda)[:, :R], refs[last][2].view(F + 1, lda)[:, :R]
        assert torch.equal(V, Vr), n


@pytest.mark.parametrize("name,size", [("c1_poisson1d", "full"), ("c2_poisson2d", "full"),
                                       ("c3_poisson5d", "mini")])
def test_cuda_graph_replay_matches_eager_calls(name, size):
    """bench.py's per_config times the bench's call replayed in CUDA graphs of 10 steps (the
    fused single launch for C1, the two launches with programmatic dependent launch for C2/C3):
    a captured sequence alternating seeds and rhs values into ONE [A | b] (and a second buffer)
    leaves, after every replay, exactly the bits of the eager calls -- the last call's in the
    shared buffer"""
    p = wl.make_problem(name, size)
    d, F, R = p.dim, p.n_features, p.n_rows
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ctx = fls.Context(stream=s)
        base = dev_blocks(p)
        alt = [fls.Block(b.X, b.terms, b.weight, 2.0 * b.values - 1.0, b.fields) for b in base]
        sets = [fls.BlockSet(base, d), fls.BlockSet(alt, d)]
        lda = fls.round_up(R, 4)
        refs = []
        for k in range(2):
            W, b, A, _ = fls.fls_features_assemble(ctx, d, F, p.sigma, k, sets[k], lda=lda)
            fls.fls_sync(ctx)
            refs.append((W.clone(), b.clone(), A[: (F + 1) * lda].view(F + 1, lda)[:, :R].clone()))
        A = torch.full(((F + 1) * lda,), float("nan"), dtype=torch.float64, device="cuda")
        A2 = torch.full_like(A, float("nan"))
        W = torch.empty((F, d), dtype=torch.float64, device="cuda")
        b = torch.empty((F,), dtype=torch.float64, device="cuda")
        W2, b2 = torch.empty_like(W), torch.empty_like(b)

        def seq():
            for i in range(5):                       # seeds 0, 1, 0, 1, 0: ends on seed 0
                fls.fls_features_assemble(ctx, d, F, p.sigma, i % 2, sets[i % 2],
                                          W=W, b=b, A=A, lda=lda)
            fls.fls_features_assemble(ctx, d, F, p.sigma, 1, sets[1], W=W2, b=b2, A=A2, lda=lda)

        seq()                                        # warm-up outside the capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            seq()
        for rep in range(3):
            A.fill_(float("nan"))
            A2.fill_(float("nan"))
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(W, refs[0][0]) and torch.equal(b, refs[0][1]), rep
            assert torch.equal(A.view(F + 1, lda)[:, :R], refs[0][2]), rep
            assert torch.equal(W2, refs[1][0]) and torch.equal(b2, refs[1][1]), rep
            assert torch.equal(A2.view(F + 1, lda)[:, :R], refs[1][2]), rep
        fls.fls_sync(ctx)
        ctx.close()


def test_concurrent_contexts_on_two_threads():
    """fls.h: calls on different contexts / streams are thread-safe -- two host threads, each
    with its own ctx on its own stream, issue interleaved fused and two-launch calls (the host
    plan state is thread-local; ctypes releases the GIL) and every buffer ends with the bits of
    the same call made alone"""
    import threading
    probs = [wl.make_problem("c1_poisson1d", "full"), wl.make_problem("c2_poisson2d", "full")]
    refs, setups = [], []
    for p in probs:
        d, F, R = p.dim, p.n_features, p.n_rows
        s = torch.cuda.Stream()
        ctx = fls.Context(stream=s)
        bs = fls.BlockSet(dev_blocks(p), d)
        lda = fls.round_up(R, 4)
        with torch.cuda.stream(s):
            W, b, A, _ = fls.fls_features_assemble(ctx, d, F, p.sigma, 3, bs, lda=lda)
        fls.fls_sync(ctx)
        refs.append((W.clone(), b.clone(), A.view(F + 1, lda)[:, :R].clone()))
        setups.append((p, s, ctx, bs, lda))
    outs = [None, None]
    errs = []

    def work(k):
        try:
            p, s, ctx, bs, lda = setups[k]
            d, F = p.dim, p.n_features
            W = torch.empty((F, d), dtype=torch.float64, device="cuda")
            b = torch.empty((F,), dtype=torch.float64, device="cuda")
            A = torch.full((((F + 1) * lda),), float("nan"), dtype=torch.float64, device="cuda")
            with torch.cuda.stream(s):
                for i in range(20):
                    fls.fls_features_assemble(ctx, d, F, p.sigma, 3 if i % 2 == 1 else 5, bs,
                                              W=W, b=b, A=A, lda=lda)
            fls.fls_sync(ctx)
            outs[k] = (W, b, A)
        except Exception as ex:  # noqa: BLE001
            errs.append(ex)

    th = [threading.Thread(target=work, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for k, (p, s, ctx, bs, lda) in enumerate(setups):
        F, R = p.n_features, p.n_rows
        W, b, A = outs[k]
        assert torch.equal(W, refs[k][0]) and torch.equal(b, refs[k][1]), k
        assert torch.equal(A.view(F + 1, lda)[:, :R], refs[k][2]), k
        ctx.close()


def test_maximum_operator_sizes(ctx):
    """the limits of the ABI at once: d = 8 (FLS_MAX_DIM), 64 terms (FLS_MAX_TERMS), 4 coefficient
    fields (FLS_MAX_FIELDS), and terms of order > 22 whose monomial the fold multiplies out
    axis by axis instead of from the host-expanded factor list -- vs the oracle, both folds
    (constant coefficients and per-field)"""
    g = np.random.default_rng(11)
    d, n_fields = 8, 4
    terms = []
    for t in range(64):
        alpha = [0] * d
        if t == 0:
            alpha = [3, 3, 3, 3, 3, 3, 3, 3]          # order 24 > kMaxFac
        elif t == 1:
            alpha = [0, 0, 0, 0, 0, 0, 0, 26]          # order 26 on one axis
        else:
            for _ in range(int(g.integers(0, 5))):
                alpha[int(g.integers(0, d))] += 1
        field = int(g.integers(-1, n_fields)) if t > 1 else -1
        terms.append((tuple(alpha), float(g.normal()), field))
    fields = g.uniform(0.5, 1.5, (501, n_fields))
    g2 = np.random.default_rng(12)
    W = g2.normal(0, 0.9, (97, d))                     # |W| < ~3: |W|^26 stays finite
    b = g2.uniform(0, 2 * math.pi, 97)
    X = g2.random((501, d)) * 0.5

    class B:
        pass
    h = B()
    h.X, h.terms, h.weight, h.values, h.fields = X, terms, 2.0, g2.normal(size=501), fields
    dv = fls.Block(torch.from_numpy(X).cuda(), terms, 2.0, torch.from_numpy(h.values).cuda(),
                   torch.from_numpy(fields).cuda())
    Ab, lda = fls.fls_assemble(ctx, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(), [dv])
    fls.fls_sync(ctx)
    Ao, ro, S = oracle.assemble(W, b, [h])
    Ag, rg = rows_from_colmajor(Ab, lda, 97, np.arange(501))
    emax, _ = scaled_err(Ag, Ao, S)
    assert emax <= ENTRY_TOL, emax
    assert np.array_equal(rg, ro)
    # the same operator with constant coefficients only (amplitude/phase fold path)
    const = [(a, c, -1) for a, c, _ in terms]
    h.terms, h.fields = const, None
    dv = fls.Block(torch.from_numpy(X).cuda(), const, 2.0, torch.from_numpy(h.values).cuda())
    Ab, lda = fls.fls_assemble(ctx, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(), [dv])
    fls.fls_sync(ctx)
    Ao, ro, S = oracle.assemble(W, b, [h])
    Ag, rg = rows_from_colmajor(Ab, lda, 97, np.arange(501))
    assert scaled_err(Ag, Ao, S)[0] <= ENTRY_TOL


@pytest.mark.parametrize("name", wl.CONFIG_NAMES)
def test_entries_against_long_double_truth(ctx, name):
    """both fp64 paths against the long-double truth mode on sampled rows
    of the reduced configs: the GPU entries within the 1e-12 bar of the A14 scale, and the
    oracle (the parity reference) an order of magnitude closer still"""
    p = wl.make_problem(name, "mini")
    W, b = p.parity_features()
    F = p.n_features
    Ab, lda = fls.fls_assemble(ctx, torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda(),
                               fls.BlockSet(dev_blocks(p), p.dim))
    fls.fls_sync(ctx)
    rows = np.unique(np.linspace(0, p.n_rows - 1, 24).astype(np.int64))
    Ag, _ = rows_from_colmajor(Ab, lda, F, rows)
    Ao, _, S = oracle.assemble(W, b, p.blocks, rows=rows)
    At = oracle.assemble_truth(W, b, p.blocks, rows=rows)
    e_gpu, _ = scaled_err(Ag, At, S)
    e_orc, _ = scaled_err(Ao, At, S)
    assert e_gpu <= ENTRY_TOL, e_gpu
    assert e_orc <= 2e-14, e_orc
