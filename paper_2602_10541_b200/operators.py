"""Linear differential operators as data: lists of (multi-index alpha, coefficient, field) terms
("any multi-index alpha"; P:L118 linear PDE L[u] = f; P:L402-403 variable coefficients).

These are the `terms` of fls.Block and the `fls_operator` of the C ABI.  field = -1 is a
constant coefficient; field = g >= 0 multiplies the term by coef_fields[:, g] at each point.
Time-dependent problems put time on the LAST axis (SPEC S:L153 convention).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

Term = Tuple[Tuple[int, ...], float, int]


def identity(d: int, coef: float = 1.0, field: int = -1) -> List[Term]:
    """u -> coef * u  (Dirichlet BC / IC rows, zeroth-order terms)"""
    return [(tuple([0] * d), float(coef), int(field))]


def partial(d: int, axis: int, order: int = 1, coef: float = 1.0, field: int = -1) -> List[Term]:
    """coef * d^order u / dx_axis^order"""
    if not 0 <= axis < d or order < 0:
        raise ValueError("axis / order out of range")
    a = [0] * d
    a[axis] = order
    return [(tuple(a), float(coef), int(field))]


def laplacian(d: int, coef: float = 1.0, axes: Sequence[int] = None) -> List[Term]:
    """coef * sum_k d^2/dx_k^2 over `axes` (all by default): Cor. 1, Lap phi = -|W|^2 phi"""
    axes = range(d) if axes is None else axes
    out: List[Term] = []
    for k in axes:
        out += partial(d, k, 2, coef)
    return out


def biharmonic(d: int, coef: float = 1.0) -> List[Term]:
    """coef * Lap^2 = sum_k d^4/dx_k^4 + 2 sum_{k<l} d^4/dx_k^2 dx_l^2 (Cor. 1: |W|^4 phi)"""
    out: List[Term] = []
    for k in range(d):
        out += partial(d, k, 4, coef)
    for k in range(d):
        for l in range(k + 1, d):
            a = [0] * d
            a[k] = a[l] = 2
            out.append((tuple(a), 2.0 * coef, -1))
    return out


def advection(v: Sequence[float]) -> List[Term]:
    """v . grad (Cor. 1: (v . W) cos)"""
    out: List[Term] = []
    for k, vk in enumerate(v):
        out += partial(len(v), k, 1, vk)
    return out


def helmholtz(d: int, k: float) -> List[Term]:
    """Lap + k^2 I  (prefactor (k^2 - |W|^2) on the sin cycle)"""
    return laplacian(d) + identity(d, k * k)


def heat(d_space: int, kappa: float) -> List[Term]:
    """d/dt - kappa Lap_x on (x_1..x_d, t): time is the last axis"""
    d = d_space + 1
    return partial(d, d_space, 1) + laplacian(d, -kappa, axes=range(d_space))


def wave(d_space: int, c: float) -> List[Term]:
    """d^2/dt^2 - c^2 Lap_x on (x_1..x_d, t)"""
    d = d_space + 1
    return partial(d, d_space, 2) + laplacian(d, -c * c, axes=range(d_space))


def scale(op: Sequence[Term], s: float) -> List[Term]:
    return [(a, c * s, f) for a, c, f in op]


def add(*ops: Sequence[Term]) -> List[Term]:
    out: List[Term] = []
    for op in ops:
        out += list(op)
    return out
