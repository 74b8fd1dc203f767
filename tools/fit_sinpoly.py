"""Fit the minimax polynomials used by the CUDA kernels' half-turn trig:

    sin(pi f) ~= f * p(f^2),    cos(pi f) ~= q(f^2),    f in [-1/2, 1/2].

Remez exchange on the ABSOLUTE error, all arithmetic in numpy longdouble (x87 80-bit,
Gaussian elimination written out since numpy.linalg has no longdouble), then the
coefficients are rounded to fp64 and the fp64 Horner evaluation (with fma) is checked on a
dense grid against longdouble sin / cos.  Product-side constant generator: the oracle never
uses it (it calls libm sin / cos term by term).

usage: python tools/fit_sinpoly.py NCOEF {sin|cos}
"""
import math
import sys

import numpy as np

LD = np.longdouble
PI = LD("3.14159265358979323846264338327950288")


def target(f, odd):
    return np.sin(PI * f) if odd else np.cos(PI * f)


def basis(f, j, odd):
    return f ** (2 * j + 1) if odd else f ** (2 * j)


def solve_ld(M, r):
    M = M.copy()
    r = r.copy()
    n = len(r)
    for k in range(n):
        piv = k + int(np.argmax(np.abs(M[k:, k])))
        M[[k, piv]] = M[[piv, k]]
        r[[k, piv]] = r[[piv, k]]
        for i in range(k + 1, n):
            m = M[i, k] / M[k, k]
            M[i, k:] -= m * M[k, k:]
            r[i] -= m * r[k]
    x = np.zeros(n, dtype=LD)
    for i in range(n - 1, -1, -1):
        x[i] = (r[i] - (M[i, i + 1:] * x[i + 1:]).sum()) / M[i, i]
    return x


def poly(c, f, odd):
    u = f * f
    p = np.zeros_like(f) + c[-1]
    for cj in c[-2::-1]:
        p = p * u + cj
    return f * p if odd else p


def remez(n, odd, iters=40):
    grid = np.linspace(LD(0), LD(0.5), 400001, dtype=LD)
    if odd:
        grid = grid[1:]
    k = np.arange(n + 1)
    ref = LD(0.25) * (1 - np.cos(PI * LD(1) * (k.astype(LD) + (1 if odd else 0)) / (n + (1 if odd else 0))))
    ref = np.clip(ref, grid[0], LD(0.5))
    best = None
    for _ in range(iters):
        M = np.zeros((n + 1, n + 1), dtype=LD)
        for i, f in enumerate(ref):
            for j in range(n):
                M[i, j] = basis(f, j, odd)
            M[i, n] = LD((-1) ** i)
        sol = solve_ld(M, target(ref, odd))
        c = sol[:n]
        err = poly(c, grid, odd) - target(grid, odd)
        emax = np.abs(err).max()
        if best is None or emax < best[1]:
            best = (c, emax)
        s = np.sign(err)
        cuts = np.flatnonzero(s[1:] != s[:-1]) + 1
        segs = np.split(np.arange(grid.size), cuts)
        ext = np.array([seg[np.argmax(np.abs(err[seg]))] for seg in segs if seg.size])
        if ext.size < n + 1:
            break
        if ext.size > n + 1:   # keep the n+1 consecutive extrema with the largest minimum
            mags = np.abs(err[ext])
            starts = range(ext.size - n)
            st = max(starts, key=lambda a: mags[a:a + n + 1].min())
            ext = ext[st:st + n + 1]
        ref = grid[ext]
    return best


def check_fp64(c64, odd):
    f = np.linspace(-0.5, 0.5, 2000001)
    u = f * f
    p = np.full_like(f, c64[-1])
    for cj in c64[-2::-1]:
        p = p * u + cj
    y = f * p if odd else p
    return float(np.abs(y.astype(LD) - target(f.astype(LD), odd)).max())


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 7
    odd = (sys.argv[2] if len(sys.argv) > 2 else "sin") == "sin"
    c, e = remez(n, odd)
    c64 = np.array([float(x) for x in c])
    deg = 2 * n - 1 if odd else 2 * n - 2
    print(f"{'sin' if odd else 'cos'} ncoef={n} degree={deg} remez max abs err (longdouble) = {float(e):.3e}")
    print(f"fp64-rounded coefficients, fp64 Horner: max abs err = {check_fp64(c64, odd):.3e}")
    for j, x in enumerate(c64):
        print(f"  c{j} = {float(x).hex()}  /* {float(x)!r} */")
