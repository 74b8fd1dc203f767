"""The shared input generator (workloads/): manufactured sources, point placement, shapes.

pins: finite differences of u* (brute force) for every config's f = L u*; the
on-face / initial-slab invariants; row counts of BASELINE.json.
"""
import numpy as np
import pytest

import workloads as wl


def _apply_fd(u, X, terms, fields=None, h=1e-3):
    """L u at X by central differences (orders <= 4, one axis per term or (2,2) mixes)."""
    d = X.shape[1]
    out = np.zeros(X.shape[0])
    st = {0: [(0, 1.0)], 1: [(-1, -0.5), (1, 0.5)], 2: [(-1, 1.0), (0, -2.0), (1, 1.0)],
          4: [(-2, 1.0), (-1, -4.0), (0, 6.0), (1, -4.0), (2, 1.0)]}
    import itertools
    for alpha, coef, field in terms:
        acc = np.zeros(X.shape[0])
        for combo in itertools.product(*[st[a] for a in alpha]):
            off = np.array([o for o, _ in combo], float) * h
            w = np.prod([c for _, c in combo]) / h ** sum(alpha)
            acc += w * u(X + off)
        c = coef * (fields[:, field] if field >= 0 else 1.0)
        out += c * acc
    return out


@pytest.mark.parametrize("name", wl.CONFIG_NAMES)
def test_manufactured_source_matches_fd(name):
    p = wl.make_problem(name, "mini")
    pde = p.blocks[0]
    X = pde.X[:50]
    h = 2e-3 if name == "c5_biharm3d" else 1e-4
    fd = _apply_fd(p.u_star, X, pde.terms, pde.fields[:50] if pde.fields is not None else None, h)
    rel = np.abs(fd - pde.values[:50]).max() / np.abs(pde.values[:50]).max()
    assert rel < (1e-4 if name == "c5_biharm3d" else 1e-6), rel


@pytest.mark.parametrize("name", wl.CONFIG_NAMES)
def test_bc_values_and_placement(name):
    p = wl.make_problem(name, "mini")
    lo, hi = p.lo, p.hi
    for blk in p.blocks:
        assert blk.X.flags.c_contiguous and blk.X.dtype == np.float64
        assert np.all(blk.X >= lo - 1e-15) and np.all(blk.X <= hi + 1e-15)
        if blk.name == "bc":
            on_face = np.any((blk.X == lo) | (blk.X == hi), axis=1)
            assert on_face.all()
            assert np.array_equal(blk.values, p.u_star(blk.X))
        if blk.name == "ic":
            assert np.all(blk.X[:, -1] == 0.0)
            assert np.array_equal(blk.values, p.u_star(blk.X))


def test_full_row_counts_match_baseline():
    # BASELINE.json configs: R = 1,002 / 4,800 / 25,000 / 65,000 / 2,097,152 (C5 not built here)
    exp = {"c1_poisson1d": (1002, 500), "c2_poisson2d": (4800, 2000),
           "c3_poisson5d": (25000, 4000), "c4_heat2d": (65000, 8000)}
    for name, (R, F) in exp.items():
        p = wl.make_problem(name, "full")
        assert p.n_rows == R and p.n_features == F
    assert wl.FULL["c5_biharm3d"] == dict(n_int=2_097_152, n_features=8192)


def test_determinism_and_shards():
    a = wl.make_problem("c3_poisson5d", "mini")
    b = wl.make_problem("c3_poisson5d", "mini")
    for x, y in zip(a.blocks, b.blocks):
        assert x.X.tobytes() == y.X.tobytes()
    R = 1002
    for P in (1, 2, 3, 8):
        spans = [wl.shard_range(R, r, P) for r in range(P)]
        assert spans[0][0] == 0 and spans[-1][1] == R
        assert all(spans[i][1] == spans[i + 1][0] for i in range(P - 1))
    rows = wl.sample_rows(2_097_152)
    assert rows[0] == 0 and rows[-1] == 2_097_151 and np.all(np.diff(rows) > 0)
