"""Fit the odd minimax polynomial  sin(pi*f) ~= f * p(f^2),  f in [-1/2, 1/2],
used by the CUDA assembly kernel's half-turn range reduction.

Remez exchange on the ABSOLUTE error in numpy longdouble (x87 80-bit), then the
coefficients are rounded to fp64 and the fp64 Horner evaluation is checked on a
dense grid against longdouble sin.  Product-side constant generator: the oracle
never uses it (it calls libm sin/cos term by term).

usage: python tools/fit_sinpoly.py [ncoef]
"""
import sys
import numpy as np

LD = np.longdouble
PI = LD("3.14159265358979323846264338327950288")


def remez_odd(ncoef, iters=60):
    # unknowns: c_0..c_{n-1}, E ; equations at n+1 reference points in (0, 1/2]
    n = ncoef
    k = np.arange(n + 1, dtype=LD)
    # Chebyshev-like initial reference on (0, 0.5]
    ref = LD(0.25) * (1 - np.cos(PI * (k + 1) / (n + 1)))
    ref = ref / ref.max() * LD(0.5)
    grid = np.linspace(LD(1e-6), LD(0.5), 200001, dtype=LD)
    for _ in range(iters):
        M = np.zeros((n + 1, n + 1), dtype=LD)
        for i, f in enumerate(ref):
            for j in range(n):
                M[i, j] = f ** (2 * j + 1)
            M[i, n] = (-1) ** i
        rhs = np.sin(PI * ref)
        # solve in float64 then refine in longdouble (numpy.linalg lacks longdouble)
        sol = np.linalg.solve(M.astype(np.float64), rhs.astype(np.float64)).astype(LD)
        for _r in range(3):
            res = rhs - M @ sol
            sol = sol + np.linalg.solve(M.astype(np.float64), res.astype(np.float64)).astype(LD)
        c = sol[:n]
        err = poly(c, grid) - np.sin(PI * grid)
        # new reference: extrema of err, one per sign-alternating segment
        s = np.sign(err)
        idx = np.flatnonzero(np.diff(s) != 0)
        segs = np.split(np.arange(grid.size), idx + 1)
        ext = [seg[np.argmax(np.abs(err[seg]))] for seg in segs]
        if len(ext) < n + 1:
            break
        # keep n+1 largest-alternating: take the last n+1 (includes f=0.5 end)
        ext = ext[-(n + 1):]
        ref = grid[ext]
    return c, np.abs(err).max()


def poly(c, f):
    u = f * f
    p = np.zeros_like(f) + c[-1]
    for cj in c[-2::-1]:
        p = p * u + cj
    return f * p


def check_fp64(c64):
    f = np.linspace(-0.5, 0.5, 2000001)
    u = f * f
    p = np.full_like(f, c64[-1])
    for cj in c64[-2::-1]:
        p = p * u + cj  # numpy: separate mul+add (kernel uses fma: at least as accurate)
    y = f * p
    ref = np.sin(PI * f.astype(LD))
    return float(np.abs(y.astype(LD) - ref).max())


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 7
    c, e = remez_odd(n)
    c64 = np.array([float(x) for x in c])
    print(f"ncoef={n} degree={2*n-1} remez max abs err (longdouble) = {float(e):.3e}")
    print(f"fp64-rounded coefficients, fp64 Horner: max abs err = {check_fp64(c64):.3e}")
    for j, x in enumerate(c64):
        print(f"  c{j} = {x!r}   // {x.hex()}")
