"""paper_2602_10541_b200.operators: the user-facing operator constructors (CPU, no GPU).

pins: each constructor's term list, pushed through the ORACLE's term-by-term assembly, gives
the closed forms of Cor. 1 / App. F with numpy sin / cos -- so a wrong
multi-index, coefficient or multiplicity in a constructor fails here."""
import math

import numpy as np

import oracle
from paper_2602_10541_b200 import operators as ops


class Blk:
    def __init__(self, X, terms):
        self.X, self.terms, self.weight, self.values, self.fields = X, terms, 1.0, None, None


def _A(W, b, X, terms):
    A, _, S = oracle.assemble(W, b, [Blk(X, terms)], normalize=False)
    return A, S


def test_constructors_closed_forms():
    g = np.random.default_rng(0)
    for d in (1, 2, 3, 4):
        W = g.normal(0, 2, (30, d))
        b = g.uniform(0, 2 * math.pi, 30)
        X = g.random((20, d))
        Z = X @ W.T + b
        w2 = (W ** 2).sum(1)
        for terms, ref in [(ops.identity(d, 3.0), 3.0 * np.sin(Z)),
                           (ops.laplacian(d), -w2 * np.sin(Z)),
                           (ops.biharmonic(d), w2 ** 2 * np.sin(Z)),
                           (ops.helmholtz(d, 7.0), (49.0 - w2) * np.sin(Z)),
                           (ops.advection(np.arange(1, d + 1) * 0.5), (W @ (np.arange(1, d + 1) * 0.5)) * np.cos(Z)),
                           (ops.scale(ops.laplacian(d), -2.0), 2 * w2 * np.sin(Z))]:
            A, S = _A(W, b, X, terms)
            assert np.abs(A - ref).max() <= 1e-13 * S.max()


def test_space_time_operators():
    g = np.random.default_rng(1)
    W = g.normal(0, 2, (25, 3))                       # (x, y, t)
    b = g.uniform(0, 2 * math.pi, 25)
    X = g.random((15, 3))
    Z = X @ W.T + b
    wx2 = W[:, 0] ** 2 + W[:, 1] ** 2
    A, S = _A(W, b, X, ops.heat(2, 0.1))              # u_t - 0.1 Lap_x u
    assert np.abs(A - (W[:, 2] * np.cos(Z) + 0.1 * wx2 * np.sin(Z))).max() <= 1e-13 * S.max()
    A, S = _A(W, b, X, ops.wave(2, 1.5))              # u_tt - c^2 Lap_x u
    assert np.abs(A - ((-W[:, 2] ** 2 + 2.25 * wx2) * np.sin(Z))).max() <= 1e-13 * S.max()


def test_add_and_partial_validation():
    import pytest
    assert ops.add(ops.identity(2), ops.partial(2, 1, 3)) == [((0, 0), 1.0, -1), ((0, 3), 1.0, -1)]
    with pytest.raises(ValueError):
        ops.partial(2, 2, 1)
