"""Seeded synthetic workloads for the Fast-LSQ assembly path (BASELINE.json configs 1-5).

This module is the ONE piece shared by the oracle side and the CUDA side: it produces
inputs only -- collocation points, random-feature draws for parity tests, operator term
lists, coefficient fields and manufactured right-hand sides.  It holds none of the
method's arithmetic (no derivative cycle, no monomial prefactor, no trig of a feature
phase, no least squares).  DESIGN.md §3 states the recipe; readings A3-A13 of
SURVEY.md §8(c) are the ones implemented here.

Random streams: numpy.random.Philox keyed (seed, stream_id) -- stream 1/2 are reserved
for fls_features (W / b), 3 interior, 4 boundary, 5 initial, 6 held-out test,
7 the parity-test feature draw (W ~ N(0, sigma^2), b ~ U[0, 2 pi) via numpy's own
samplers, deliberately NOT the fls_features recipe so the two never share arithmetic).
"""
from __future__ import annotations

import dataclasses
import math
from typing import Callable, List, Optional, Sequence, Tuple

import numpy as np

PI = math.pi

STREAM_FEAT_W, STREAM_FEAT_B = 1, 2
STREAM_INTERIOR, STREAM_BOUNDARY, STREAM_INITIAL, STREAM_TEST, STREAM_PARITY_FEAT = 3, 4, 5, 6, 7


def rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=int(seed) + (int(stream) << 64)))


# --------------------------------------------------------------------------------------
# operators as data: list of (alpha, coef, field)   ("multi-index alpha")
# --------------------------------------------------------------------------------------
Term = Tuple[Tuple[int, ...], float, int]   # (alpha, coef, field: -1 const / g >= 0)


def op_identity(d: int, coef: float = 1.0) -> List[Term]:
    return [(tuple([0] * d), coef, -1)]


def op_partial(d: int, axis: int, order: int, coef: float = 1.0, field: int = -1) -> List[Term]:
    a = [0] * d
    a[axis] = order
    return [(tuple(a), coef, field)]


def op_laplacian(d: int, coef: float = 1.0, axes: Optional[Sequence[int]] = None) -> List[Term]:
    axes = range(d) if axes is None else axes
    out: List[Term] = []
    for k in axes:
        out += op_partial(d, k, 2, coef)
    return out


def op_biharmonic(d: int, coef: float = 1.0) -> List[Term]:
    """Delta^2 = sum_k d^4/dx_k^4 + 2 sum_{k<l} d^4/dx_k^2 dx_l^2 (expanded)."""
    out: List[Term] = []
    for k in range(d):
        out += op_partial(d, k, 4, coef)
    for k in range(d):
        for l in range(k + 1, d):
            a = [0] * d
            a[k] = 2
            a[l] = 2
            out.append((tuple(a), 2.0 * coef, -1))
    return out


def op_advection(v: Sequence[float]) -> List[Term]:
    d = len(v)
    out: List[Term] = []
    for k in range(d):
        out += op_partial(d, k, 1, float(v[k]))
    return out


# --------------------------------------------------------------------------------------
# row blocks and configs
# --------------------------------------------------------------------------------------
@dataclasses.dataclass
class Block:
    name: str                       # "pde" | "bc" | "ic"
    X: np.ndarray                   # (n, d) float64, C-contiguous
    terms: List[Term]
    weight: float
    values: np.ndarray              # (n,) rhs values f / g / h
    fields: Optional[np.ndarray] = None   # (n, G) coefficient fields or None

    @property
    def n(self) -> int:
        return int(self.X.shape[0])


@dataclasses.dataclass
class Problem:
    name: str
    dim: int
    n_features: int
    sigma: float
    blocks: List[Block]
    u_star: Callable[[np.ndarray], np.ndarray]
    lo: np.ndarray
    hi: np.ndarray
    ridge_rel: float = 0.0          # tau = 0 for C1-C4, 1e-10 for C5
    seed: int = 0

    @property
    def n_rows(self) -> int:
        return sum(b.n for b in self.blocks)

    def block_offsets(self) -> List[int]:
        off, out = 0, []
        for b in self.blocks:
            out.append(off)
            off += b.n
        return out

    def parity_features(self) -> Tuple[np.ndarray, np.ndarray]:
        """W (F, d) ~ N(0, sigma^2), b (F,) ~ U[0, 2pi) from numpy's samplers (stream 7)."""
        g = rng(self.seed, STREAM_PARITY_FEAT)
        W = g.normal(0.0, self.sigma, size=(self.n_features, self.dim))
        b = g.uniform(0.0, 2.0 * PI, size=self.n_features)
        return np.ascontiguousarray(W), np.ascontiguousarray(b)

    def test_points(self, n: int = 10_000) -> np.ndarray:
        g = rng(self.seed, STREAM_TEST)
        return np.ascontiguousarray(self.lo + (self.hi - self.lo) * g.random((n, self.dim)))


def _uniform_box(g, n, lo, hi):
    lo = np.asarray(lo, float)
    hi = np.asarray(hi, float)
    return lo + (hi - lo) * g.random((n, lo.size))


def _faces(g, d, per_face, lo, hi, axes):
    """per_face points on each face x_k = lo_k then x_k = hi_k for k in axes (reading A5)."""
    out = []
    for k in axes:
        for v in (lo[k], hi[k]):
            P = _uniform_box(g, per_face, lo, hi)
            P[:, k] = v
            out.append(P)
    return np.concatenate(out, axis=0) if out else np.zeros((0, d))


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# manufactured solutions and their sources (verified by FD in tests/test_workloads.py)
def _u1(X):
    x = X[:, 0]
    return np.sin(3 * PI * x) + 0.5 * x * x


def _f1(X):            # -u''
    x = X[:, 0]
    return 9 * PI * PI * np.sin(3 * PI * x) - 1.0


def _u2(X):
    x, y = X[:, 0], X[:, 1]
    return np.sin(2 * PI * x) * np.sin(3 * PI * y) + np.exp(x * y)


def _f2(X):            # -Lap u
    x, y = X[:, 0], X[:, 1]
    return 13 * PI * PI * np.sin(2 * PI * x) * np.sin(3 * PI * y) - (x * x + y * y) * np.exp(x * y)


def _u3(X):
    return sum(np.sin(PI * X[:, k]) * np.cos(PI * X[:, (k + 1) % 5]) for k in range(5))


def _f3(X):            # -Lap u = 2 pi^2 u
    return 2 * PI * PI * _u3(X)


def _u4(X):            # (x, y, t), time last (reading A9)
    x, y, t = X[:, 0], X[:, 1], X[:, 2]
    return np.exp(-t) * np.sin(PI * x) * np.sin(PI * y)


def _f4(X):            # u_t - 0.1 Lap u = (0.2 pi^2 - 1) u
    return (0.2 * PI * PI - 1.0) * _u4(X)


def _u5(X):
    return np.sin(PI * X[:, 0]) * np.sin(PI * X[:, 1]) * np.sin(PI * X[:, 2])


def _c5(X):            # variable coefficient c(x) = 1 + x_1 (reading A11)
    return 1.0 + X[:, 0]


def _f5(X):            # Lap^2 u + 16 c(x) u = (9 pi^4 + 16 (1 + x_1)) u
    return (9 * PI ** 4 + 16.0 * _c5(X)) * _u5(X)


CONFIG_NAMES = ["c1_poisson1d", "c2_poisson2d", "c3_poisson5d", "c4_heat2d", "c5_biharm3d"]

# full sizes (BASELINE.json configs 1..5)
FULL = {
    "c1_poisson1d": dict(n_int=1000, n_features=500),
    "c2_poisson2d": dict(n_int=4000, per_edge=200, n_features=2000),
    "c3_poisson5d": dict(n_int=20000, per_face=500, n_features=4000),
    "c4_heat2d": dict(n_int=50000, per_face=2500, n_ic=5000, n_features=8000),
    "c5_biharm3d": dict(n_int=2_097_152, n_features=8192),
}

# reduced sizes: the oracle finishes in about a second, still several CUDA tiles plus a ragged tail
MINI = {
    "c1_poisson1d": dict(n_int=1000, n_features=500),
    "c2_poisson2d": dict(n_int=1203, per_edge=50, n_features=333),
    "c3_poisson5d": dict(n_int=1501, per_face=37, n_features=301),
    "c4_heat2d": dict(n_int=1499, per_face=61, n_ic=157, n_features=397),
    "c5_biharm3d": dict(n_int=2049, n_features=263),
}


def make_problem(name: str, size: str = "full", seed: int = 0, **override) -> Problem:
    kw = dict((FULL if size == "full" else MINI)[name])
    kw.update(override)
    gi, gb, g0 = rng(seed, STREAM_INTERIOR), rng(seed, STREAM_BOUNDARY), rng(seed, STREAM_INITIAL)
    if name == "c1_poisson1d":
        lo, hi = np.array([-1.0]), np.array([1.0])
        Xi = _uniform_box(gi, kw["n_int"], lo, hi)
        Xb = np.array([[-1.0], [1.0]])
        blocks = [Block("pde", _c(Xi), op_laplacian(1, -1.0), 1.0, _c(_f1(Xi))),
                  Block("bc", _c(Xb), op_identity(1), 10.0, _c(_u1(Xb)))]
        return Problem(name, 1, kw["n_features"], 10.0, blocks, _u1, lo, hi, 0.0, seed)
    if name == "c2_poisson2d":
        lo, hi = np.zeros(2), np.ones(2)
        Xi = _uniform_box(gi, kw["n_int"], lo, hi)
        # edges y=0, y=1, x=0, x=1 (reading A5)
        Xb = _faces(gb, 2, kw["per_edge"], lo, hi, axes=[1, 0])
        blocks = [Block("pde", _c(Xi), op_laplacian(2, -1.0), 1.0, _c(_f2(Xi))),
                  Block("bc", _c(Xb), op_identity(2), 100.0, _c(_u2(Xb)))]
        return Problem(name, 2, kw["n_features"], 5.0, blocks, _u2, lo, hi, 0.0, seed)
    if name == "c3_poisson5d":
        lo, hi = np.zeros(5), np.ones(5)
        Xi = _uniform_box(gi, kw["n_int"], lo, hi)
        Xb = _faces(gb, 5, kw["per_face"], lo, hi, axes=range(5))
        blocks = [Block("pde", _c(Xi), op_laplacian(5, -1.0), 1.0, _c(_f3(Xi))),
                  Block("bc", _c(Xb), op_identity(5), 100.0, _c(_u3(Xb)))]
        return Problem(name, 5, kw["n_features"], 2.0, blocks, _u3, lo, hi, 0.0, seed)
    if name == "c4_heat2d":
        lo, hi = np.zeros(3), np.ones(3)
        Xi = _uniform_box(gi, kw["n_int"], lo, hi)
        Xb = _faces(gb, 3, kw["per_face"], lo, hi, axes=[0, 1])      # lateral faces only
        X0 = _uniform_box(g0, kw["n_ic"], lo, hi)
        X0[:, 2] = 0.0
        heat = op_partial(3, 2, 1, 1.0) + op_laplacian(3, -0.1, axes=[0, 1])
        blocks = [Block("pde", _c(Xi), heat, 1.0, _c(_f4(Xi))),
                  Block("bc", _c(Xb), op_identity(3), 100.0, _c(_u4(Xb))),
                  Block("ic", _c(X0), op_identity(3), 100.0, _c(_u4(X0)))]
        return Problem(name, 3, kw["n_features"], 4.0, blocks, _u4, lo, hi, 0.0, seed)
    if name == "c5_biharm3d":
        lo, hi = np.zeros(3), np.ones(3)
        Xi = _uniform_box(gi, kw["n_int"], lo, hi)
        terms = op_biharmonic(3, 1.0) + [((0, 0, 0), 16.0, 0)]       # reading A11
        blocks = [Block("pde", _c(Xi), terms, 1.0, _c(_f5(Xi)), fields=_c(_c5(Xi)[:, None]))]
        return Problem(name, 3, kw["n_features"], 3.0, blocks, _u5, lo, hi, 1e-10, seed)
    raise KeyError(name)


# --------------------------------------------------------------------------------------
# nonlinear problems for the Newton path.  L[u] + N(u) = f with a
# pointwise N, Dirichlet rows weighted by lambda = 100.  The paper's own nonlinear
# benchmarks (Table 2) state no manufactured solutions; these are synthetic stand-ins of the
# same form (NL-Poisson u^3 term, Bratu exponential term).
# --------------------------------------------------------------------------------------
def _u_nl(X):
    x, y = X[:, 0], X[:, 1]
    return np.sin(PI * x) * np.sin(PI * y) + x * y


def _u_bratu(X):
    return np.sin(PI * X[:, 0]) * np.sin(PI * X[:, 1])


NL_NAMES = ["nl_poisson2d", "bratu2d"]


def make_nl_problem(name: str, n_int: int = 1500, per_edge: int = 100, n_features: int = 400,
                    sigma: float = 3.0, seed: int = 0) -> Problem:
    gi, gb = rng(seed, STREAM_INTERIOR), rng(seed, STREAM_BOUNDARY)
    lo, hi = np.zeros(2), np.ones(2)
    Xi = _uniform_box(gi, n_int, lo, hi)
    Xb = _faces(gb, 2, per_edge, lo, hi, axes=[1, 0])
    if name == "nl_poisson2d":         # -Lap u + u^3 = f
        u = _u_nl
        f = 2 * PI * PI * np.sin(PI * Xi[:, 0]) * np.sin(PI * Xi[:, 1]) + u(Xi) ** 3
        nl = ("poly", [0.0, 0.0, 0.0, 1.0])
    elif name == "bratu2d":            # -Lap u - e^u = f  (Bratu, lambda = 1)
        u = _u_bratu
        f = 2 * PI * PI * u(Xi) - np.exp(u(Xi))
        nl = ("exp", [-1.0, 1.0])
    else:
        raise KeyError(name)
    blocks = [Block("pde", _c(Xi), op_laplacian(2, -1.0), 1.0, _c(f)),
              Block("bc", _c(Xb), op_identity(2), 100.0, _c(u(Xb)))]
    p = Problem(name, 2, n_features, sigma, blocks, u, lo, hi, 0.0, seed)
    p.nl = nl
    return p


def make_burgers1d(nu_final: float = 0.2, n_int: int = 400, n_features: int = 200,
                   sigma: float = 8.0, seed: int = 0):
    """Steady viscous Burgers  -nu u'' + u u' = 0  on [-1, 1] (the paper's continuation case,
    P:L167), Dirichlet rows u(-1) = -u(1) = tanh(1/(2 nu_final)) (lambda = 100) so that
    u* = -tanh(x / (2 nu_final)) solves the final stage exactly.  Returns (problem, make_pde):
    make_pde(nu) gives the PDE block for one continuation stage (f = 0)."""
    gi = rng(seed, STREAM_INTERIOR)
    lo, hi = np.array([-1.0]), np.array([1.0])
    Xi = _c(_uniform_box(gi, n_int, lo, hi))
    Xb = np.array([[-1.0], [1.0]])

    def u(X):
        return -np.tanh(X[:, 0] / (2.0 * nu_final))

    def make_pde(nu):
        return Block("pde", Xi, op_partial(1, 0, 2, -float(nu)), 1.0, np.zeros(n_int))
    blocks = [make_pde(nu_final), Block("bc", _c(Xb), op_identity(1), 100.0, _c(u(Xb)))]
    p = Problem("burgers1d", 1, n_features, sigma, blocks, u, lo, hi, 0.0, seed)
    p.nl = ("udu", [1.0], (1,))
    return p, make_pde


def make_helmholtz2d(n_int: int = 600, per_edge: int = 40, n_features: int = 120, k: float = 10.0,
                     seed: int = 0) -> Problem:
    """Helmholtz 2D (the paper's learnable-bandwidth demonstration case):
    Lap u + k^2 u = f on [0,1]^2, Dirichlet (lambda = 100), u* = sin(4 pi x) sin(4 pi y) (a
    synthetic stand-in: the paper states no u*).  Problem.sigma = 1 so parity_features()
    returns the frozen base weights W^ ~ N(0, I) of App. E."""
    gi, gb = rng(seed, STREAM_INTERIOR), rng(seed, STREAM_BOUNDARY)
    lo, hi = np.zeros(2), np.ones(2)
    Xi = _uniform_box(gi, n_int, lo, hi)
    Xb = _faces(gb, 2, per_edge, lo, hi, axes=[1, 0])

    def u(X):
        return np.sin(4 * PI * X[:, 0]) * np.sin(4 * PI * X[:, 1])
    f = (k * k - 32 * PI * PI) * u(Xi)
    blocks = [Block("pde", _c(Xi), op_laplacian(2, 1.0) + op_identity(2, k * k), 1.0, _c(f)),
              Block("bc", _c(Xb), op_identity(2), 100.0, _c(u(Xb)))]
    return Problem("helmholtz2d", 2, n_features, 1.0, blocks, u, lo, hi, 0.0, seed)


def make_helmholtz2d_var(n_int: int = 600, per_edge: int = 40, n_features: int = 120,
                         k: float = 10.0, seed: int = 0) -> Problem:
    """Variable-coefficient Helmholtz 2D: Lap u + k^2 (1 + x_1) u = f on [0,1]^2 (coefficient
    field c(x) = 1 + x_1 on the zeroth-order term, as in config 5's reading A11), Dirichlet
    (lambda = 100), u* = sin(4 pi x) sin(4 pi y), f = (k^2 (1 + x_1) - 32 pi^2) u*.  For the
    learnable-bandwidth gradient with coefficient fields."""
    gi, gb = rng(seed, STREAM_INTERIOR), rng(seed, STREAM_BOUNDARY)
    lo, hi = np.zeros(2), np.ones(2)
    Xi = _uniform_box(gi, n_int, lo, hi)
    Xb = _faces(gb, 2, per_edge, lo, hi, axes=[1, 0])

    def u(X):
        return np.sin(4 * PI * X[:, 0]) * np.sin(4 * PI * X[:, 1])
    cf = 1.0 + Xi[:, 0]
    f = (k * k * cf - 32 * PI * PI) * u(Xi)
    blocks = [Block("pde", _c(Xi), op_laplacian(2, 1.0) + [((0, 0), k * k, 0)], 1.0, _c(f),
                    fields=_c(cf[:, None])),
              Block("bc", _c(Xb), op_identity(2), 100.0, _c(u(Xb)))]
    return Problem("helmholtz2d_var", 2, n_features, 1.0, blocks, u, lo, hi, 0.0, seed)


def sample_rows(n_rows: int, n_shards: int = 8, stride: int = 256) -> np.ndarray:
    """Deterministic sampled global rows: every stride-th row plus the first and last
    row of every shard of an n_shards-way split."""
    rows = set(range(0, n_rows, stride))
    for r in range(n_shards):
        a, b = (r * n_rows) // n_shards, ((r + 1) * n_rows) // n_shards
        if b > a:
            rows.add(a)
            rows.add(b - 1)
    return np.array(sorted(rows), dtype=np.int64)


def shard_range(n_rows: int, rank: int, world: int) -> Tuple[int, int]:
    """Rank r owns global rows [floor(r R / P), floor((r+1) R / P))."""
    return (rank * n_rows) // world, ((rank + 1) * n_rows) // world
