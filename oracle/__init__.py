"""CPU oracle for the Fast-LSQ assembly path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.  The product path (paper_2602_10541_b200) never imports it and
shares no code with it (see oracle/oracle.c header).

ctypes wrapper over liboracle.so (plain C, gcc -O2 -ffp-contract=off -fopenmp).
Functions follow the paper's definitions; each C function cites its passage.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
ORC_MAX_DIM = 8


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-std=c11", "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Term(C.Structure):
    _fields_ = [("alpha", C.c_int32 * ORC_MAX_DIM), ("coef", C.c_double), ("field", C.c_int32)]


class _Block(C.Structure):
    _fields_ = [("X", C.c_void_p), ("n_points", C.c_int64), ("terms", C.c_void_p),
                ("n_terms", C.c_int32), ("coef_fields", C.c_void_p), ("n_fields", C.c_int32),
                ("weight", C.c_double), ("values", C.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        L.orc_philox4x64.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_raw_stream.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int64, C.c_void_p]
        L.orc_features.argtypes = [C.c_int, C.c_int64, C.c_double, C.c_uint64, C.c_void_p, C.c_void_p]
        L.orc_features_blocks.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_uint64,
                                          C.c_void_p, C.c_void_p]
        L.orc_sample_box.argtypes = [C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_uint64,
                                     C.c_uint64, C.c_void_p]
        L.orc_sample_faces.argtypes = [C.c_int, C.c_int64, C.c_uint32, C.c_void_p, C.c_void_p,
                                       C.c_uint64, C.c_uint64, C.c_void_p]
        L.orc_diff.argtypes =[C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_assemble.argtypes = [C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                   C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_assemble_truth.argtypes = [C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_int,
                                         C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.c_void_p]
        L.orc_lstsq.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_double,
                                C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_lstsq_mu.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_double,
                                   C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_eval.argtypes =[C.c_int, C.c_int64, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                               C.c_void_p, C.c_int64, C.c_void_p]
        L.orc_max_threads.restype = C.c_int
        L.orc_set_threads.argtypes = [C.c_int]
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def max_threads() -> int:
    return int(lib().orc_max_threads())


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def philox4x64(ctr: Sequence[int], key: Sequence[int]) -> np.ndarray:
    c = np.array(ctr, dtype=np.uint64)
    k = np.array(key, dtype=np.uint64)
    out = np.zeros(4, dtype=np.uint64)
    lib().orc_philox4x64(_p(c), _p(k), _p(out))
    return out


def raw_stream(seed: int, stream: int, n0: int, count: int) -> np.ndarray:
    out = np.zeros(count, dtype=np.uint64)
    lib().orc_raw_stream(seed, stream, n0, count, _p(out))
    return out


def features(dim: int, n_features: int, sigma: float, seed: int):
    W = np.zeros((n_features, dim))
    b = np.zeros(n_features)
    lib().orc_features(dim, n_features, sigma, seed, _p(W), _p(b))
    return W, b


def features_blocks(dim: int, counts: Sequence[int], sigmas: Sequence[float], seed: int):
    F = int(sum(counts))
    W = np.zeros((F, dim))
    b = np.zeros(F)
    c = np.array(counts, dtype=np.int64)
    s = np.array(sigmas, dtype=np.float64)
    lib().orc_features_blocks(dim, len(counts), _p(c), _p(s), seed, _p(W), _p(b))
    return W, b


def sample_box(dim, n, lo, hi, seed, stream):
    X = np.zeros((n, dim))
    lo = _f64(lo)
    hi = _f64(hi)
    lib().orc_sample_box(dim, n, _p(lo), _p(hi), seed, stream, _p(X))
    return X


def sample_faces(dim, per_face, axes_mask, lo, hi, seed, stream):
    nax = bin(axes_mask).count("1")
    X = np.zeros((2 * per_face * nax, dim))
    lo = _f64(lo)
    hi = _f64(hi)
    lib().orc_sample_faces(dim, per_face, axes_mask, _p(lo), _p(hi), seed, stream, _p(X))
    return X


def diff(alpha: Sequence[int]):
    """Symbolic D^alpha sin(W.x+b) -> (exponent vector e, phase p), one derivative at a time."""
    d = len(alpha)
    a = np.zeros(ORC_MAX_DIM, dtype=np.int32)
    a[:d] = alpha
    e = np.zeros(ORC_MAX_DIM, dtype=np.int32)
    p = np.zeros(1, dtype=np.int32)
    lib().orc_diff(d, _p(a), _p(e), _p(p))
    return tuple(int(v) for v in e[:d]), int(p[0])


class _BlockKeep:
    """keeps numpy buffers alive while the C structs point at them"""

    def __init__(self, blocks):
        self.keep = []
        self.arr = (_Block * len(blocks))()
        for q, blk in enumerate(blocks):
            X = _f64(blk.X)
            terms = (_Term * len(blk.terms))()
            for t, (alpha, coef, field) in enumerate(blk.terms):
                for k, v in enumerate(alpha):
                    terms[t].alpha[k] = int(v)
                terms[t].coef = float(coef)
                terms[t].field = int(field)
            vals = _f64(blk.values) if blk.values is not None else None
            flds = _f64(blk.fields) if blk.fields is not None else None
            self.keep += [X, terms, vals, flds]
            B = self.arr[q]
            B.X = X.ctypes.data
            B.n_points = X.shape[0]
            B.terms = C.addressof(terms)
            B.n_terms = len(blk.terms)
            B.coef_fields = flds.ctypes.data if flds is not None else None
            B.n_fields = flds.shape[1] if flds is not None else 0
            B.weight = float(blk.weight)
            B.values = vals.ctypes.data if vals is not None else None


def assemble(W, b, blocks, rows: Optional[np.ndarray] = None, normalize: bool = True,
             want_scale: bool = True):
    """Rows `rows` (global stacked ids; default all) of [A | rhs] and the A14 scale S_ij.

    Returns (A (n_rows, F) row-major, rhs (n_rows,), S (n_rows, F) or None)."""
    W = _f64(W)
    b = _f64(b)
    F, d = W.shape
    total = sum(blk.X.shape[0] for blk in blocks)
    rows = np.arange(total, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, np.int64)
    n = rows.size
    A = np.zeros((n, F))
    rhs = np.zeros(n)
    S = np.zeros((n, F)) if want_scale else None
    keep = _BlockKeep(blocks)
    st = lib().orc_assemble(d, F, _p(W), _p(b), int(bool(normalize)), C.addressof(keep.arr),
                            len(blocks), _p(rows), n, _p(A), _p(rhs),
                            _p(S) if S is not None else None)
    if st != 0:
        raise ValueError(f"orc_assemble status {st}")
    return A, rhs, S


def assemble_truth(W, b, blocks, rows: Optional[np.ndarray] = None, normalize: bool = True):
    """orc_assemble_truth: the definition in long double, rounded to double at the end (tiny
    inputs; the near-exact reference of SURVEY §8(c) item 6).  Returns A (n_rows, F)."""
    W = _f64(W)
    b = _f64(b)
    F, d = W.shape
    total = sum(blk.X.shape[0] for blk in blocks)
    rows = np.arange(total, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, np.int64)
    A = np.zeros((rows.size, F))
    keep = _BlockKeep(blocks)
    st = lib().orc_assemble_truth(d, F, _p(W), _p(b), int(bool(normalize)), C.addressof(keep.arr),
                                  len(blocks), _p(rows), rows.size, _p(A))
    if st != 0:
        raise ValueError(f"orc_assemble_truth status {st}")
    return A


def lstsq(A, bvec, ridge_rel: float = 0.0):
    """argmin ||A beta - b||^2 + mu ||beta||^2, sqrt(mu) = ridge_rel ||A||_F, Householder QR.

    Returns (beta, residual norm, diag(R))."""
    A = _f64(A)
    bvec = _f64(bvec)
    m, n = A.shape
    beta = np.zeros(n)
    res = np.zeros(1)
    rd = np.zeros(n)
    st = lib().orc_lstsq(_p(A), m, n, _p(bvec), float(ridge_rel), _p(beta), _p(res), _p(rd))
    if st == -3:
        raise MemoryError("orc_lstsq allocation failed")
    if st != 0:
        raise np.linalg.LinAlgError(f"orc_lstsq status {st} (zero diagonal in R)")
    return beta, float(res[0]), rd


def lstsq_mu(A, bvec, sqrt_mu: float):
    """argmin ||A beta - b||^2 + mu ||beta||^2 with an absolute sqrt(mu) (Newton step)"""
    A = _f64(A)
    bvec = _f64(bvec)
    m, n = A.shape
    beta = np.zeros(n)
    res = np.zeros(1)
    rd = np.zeros(n)
    st = lib().orc_lstsq_mu(_p(A), m, n, _p(bvec), float(sqrt_mu), _p(beta), _p(res), _p(rd))
    if st != 0:
        raise np.linalg.LinAlgError(f"orc_lstsq_mu status {st}")
    return beta, float(res[0]), rd


def evaluate(W, b, beta, X, normalize: bool = True) -> np.ndarray:
    W = _f64(W)
    b = _f64(b)
    beta = _f64(beta)
    X = _f64(X)
    F, d = W.shape
    out = np.zeros(X.shape[0])
    lib().orc_eval(d, F, _p(W), _p(b), int(bool(normalize)), _p(beta), _p(X), X.shape[0], _p(out))
    return out
