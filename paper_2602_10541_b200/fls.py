"""Thin Python binding of libfls with the C ABI's names (include/fls.h).

Argument marshalling only: torch CUDA tensors in, device pointers + sizes out to the C ABI;
every step of the path runs in libfls kernels (or cuSOLVER/cuBLAS inside fls_solve).  There
is no CPU fallback -- calling anything here without a CUDA device and a built libfls.so
raises.

    ctx = Context()                                   # borrows torch's current stream
    W, b = fls_features(ctx, dim, F, sigma, seed)
    A, rhs = fls_assemble(ctx, W, b, blocks)         # [A | rhs] column-major, lda padded
    beta, res = fls_solve(ctx, Ab, n_rows, lda, F, ridge_rel)   # destroys Ab; TSQR over the
                                                               # ranks when a comm is attached
    u = fls_eval(ctx, W, b, beta, X)
"""
from __future__ import annotations

import ctypes as C
import dataclasses
from typing import List, Optional, Sequence, Tuple

import torch

from . import _abi
from ._abi import FLS_COL_MAJOR, FLS_ROW_MAJOR, FlsError, check

Term = Tuple[Sequence[int], float, int]   # (alpha, coef, field)

__all__ = ["Context", "Block", "fls_features", "fls_assemble", "fls_features_assemble", "fls_solve",
           "fls_solve_mu", "fls_comm_unique_id", "fls_comm_init", "fls_comm_init_host",
           "fls_comm_destroy", "fls_comm_config", "fls_comm_info", "fls_qr_r",
           "fls_frob2", "fls_geqrf", "fls_solve_stacked", "fls_eval", "fls_eval_block", "fls_ipc_handle", "fls_ipc_open",
           "fls_ipc_close", "fls_sync", "fls_ctx_timing", "fls_ctx_timing_read",
           "fls_assemble_host", "HostBlockSet", "BlockSet", "fls_features_blocks", "QRFactor",
           "make_nonlinearity", "fls_nl_residual", "fls_axpy", "fls_features_transform",
           "fls_bandwidth_grad", "fls_sample_box", "fls_sample_faces", "FlsError", "FLS_COL_MAJOR", "FLS_ROW_MAJOR",
           "round_up"]


def round_up(n: int, m: int) -> int:
    return ((n + m - 1) // m) * m


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _dev_f64(t: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != torch.float64:
        raise TypeError(f"{name} must be float64")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _on(ctx: "Context", t: torch.Tensor, name: str) -> torch.Tensor:
    """t must live on the ctx's device (a kernel would otherwise read another GPU's address)"""
    if t.device.type != "cuda" or t.device.index != ctx.device:
        raise ValueError(f"{name} is on {t.device}, the ctx on cuda:{ctx.device}")
    return t


def _need(t: torch.Tensor, n: int, name: str):
    """t must hold at least n doubles (the kernels write / read that far)"""
    if t.numel() < n:
        raise ValueError(f"{name} holds {t.numel()} doubles; this call needs >= {n}")


def _basis(ctx: "Context", W: torch.Tensor, b: torch.Tensor):
    _on(ctx, _dev_f64(W, "W"), "W")
    _on(ctx, _dev_f64(b, "b"), "b")
    if W.dim() != 2:
        raise ValueError("W must be (n_features, dim)")
    F, dim = int(W.shape[0]), int(W.shape[1])
    if b.numel() != F:
        raise ValueError(f"b has {b.numel()} entries, W has {F} features")
    return F, dim


class Context:
    """fls_ctx on a device, borrowing a CUDA stream (default: torch's current stream)."""

    def __init__(self, device: Optional[int] = None, stream: Optional[torch.cuda.Stream] = None):
        lib = _abi.load()
        if not torch.cuda.is_available():
            raise FlsError(3, "no CUDA device: libfls has no CPU path")
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = C.c_void_p()
        check(lib.fls_ctx_create(self.device, C.c_void_p(self.stream.cuda_stream), C.byref(h)))
        self.handle = h

    def set_stream(self, stream: torch.cuda.Stream):
        self.stream = stream
        check(_abi.load().fls_ctx_set_stream(self.handle, C.c_void_p(stream.cuda_stream)))

    def close(self):
        if getattr(self, "handle", None):
            _abi.load().fls_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fls_sync(ctx: Context):
    check(_abi.load().fls_sync(ctx.handle))


def fls_ctx_timing(ctx: Context, enable: bool = True):
    check(_abi.load().fls_ctx_timing(ctx.handle, int(bool(enable))))


def fls_ctx_timing_read(ctx: Context):
    """(summed assembly-kernel ms, launches) since the last enable / read"""
    ms = C.c_double(0.0)
    n = C.c_int64(0)
    check(_abi.load().fls_ctx_timing_read(ctx.handle, C.byref(ms), C.byref(n)))
    return ms.value, n.value


class _Op:
    def __init__(self, dim: int, terms: Sequence[Term]):
        n = len(terms)
        self.arr = (_abi.fls_term * max(n, 1))()
        for t, (alpha, coef, field) in enumerate(terms):
            for k, v in enumerate(alpha):
                self.arr[t].alpha[k] = int(v)
            self.arr[t].coef = float(coef)
            self.arr[t].field = int(field)
        self.op = _abi.fls_operator(int(dim), n, C.cast(self.arr, C.POINTER(_abi.fls_term)))


@dataclasses.dataclass
class Block:
    """one row block of Eq. 3 (device tensors)"""
    X: torch.Tensor                      # (n, d) float64 CUDA
    terms: List[Term]
    weight: float = 1.0
    values: Optional[torch.Tensor] = None
    fields: Optional[torch.Tensor] = None   # (n, G)

    @property
    def n(self) -> int:
        return int(self.X.shape[0])


def fls_features(ctx: Context, dim: int, n_features: int, sigma: float, seed: int,
                 W: Optional[torch.Tensor] = None, b: Optional[torch.Tensor] = None):
    dev = torch.device("cuda", ctx.device)
    W = torch.empty((n_features, dim), dtype=torch.float64, device=dev) if W is None else W
    b = torch.empty((n_features,), dtype=torch.float64, device=dev) if b is None else b
    _on(ctx, _dev_f64(W, "W"), "W")
    _on(ctx, _dev_f64(b, "b"), "b")
    _need(W, int(n_features) * int(dim), "W")
    _need(b, int(n_features), "b")
    check(_abi.load().fls_features(ctx.handle, int(dim), int(n_features), float(sigma),
                                   C.c_uint64(int(seed) & (2**64 - 1)), _ptr(W), _ptr(b)))
    return W, b


def fls_features_blocks(ctx: Context, dim: int, block_features: Sequence[int],
                        sigmas: Sequence[float], seed: int):
    """multi-block basis: block q = block_features[q] features with bandwidth sigmas[q]"""
    nb = len(block_features)
    F = int(sum(block_features))
    dev = torch.device("cuda", ctx.device)
    W = torch.empty((F, dim), dtype=torch.float64, device=dev)
    b = torch.empty((F,), dtype=torch.float64, device=dev)
    cnt = (C.c_int64 * nb)(*[int(v) for v in block_features])
    sig = (C.c_double * nb)(*[float(v) for v in sigmas])
    check(_abi.load().fls_features_blocks(ctx.handle, int(dim), nb, cnt, sig,
                                          C.c_uint64(int(seed) & (2**64 - 1)), _ptr(W), _ptr(b)))
    return W, b


def make_nonlinearity(kind: str, coefs: Sequence[float]):
    """'poly': N(u) = sum_k coefs[k] u^k;  'exp': N(u) = coefs[0] exp(coefs[1] u)"""
    nl = _abi.fls_nonlinearity()
    if kind == "poly":
        nl.kind = _abi.FLS_NL_POLY
        nl.degree = len(coefs) - 1
    elif kind == "exp":
        nl.kind = _abi.FLS_NL_EXP
        nl.degree = 1
    elif kind == "udu":                 # coefs[0] * u * D^e u  (Burgers u u_x)
        nl.kind = _abi.FLS_NL_UDU
        nl.degree = 1
    else:
        raise ValueError(kind)
    for k, v in enumerate(coefs):
        nl.a[k] = float(v)
    return nl


def fls_nl_residual(ctx: Context, nl, Lu: torch.Tensor, u: torch.Tensor, f: torch.Tensor,
                    u_prev: Optional[torch.Tensor] = None, neg_res: Optional[torch.Tensor] = None,
                    dN: Optional[torch.Tensor] = None, stats: bool = True):
    """neg_res = f - Lu - N(u), dN = N'(u); returns (neg_res, dN, (sum r^2, sum u^2, sum du^2))"""
    n = int(u.numel())
    neg_res = torch.empty_like(u) if neg_res is None else neg_res
    dN = torch.empty_like(u) if dN is None else dN
    st = (C.c_double * 3)()
    check(_abi.load().fls_nl_residual(ctx.handle, C.byref(nl), n, _ptr(Lu), _ptr(u), _ptr(u_prev),
                                      _ptr(f), _ptr(neg_res), _ptr(dN), st if stats else None))
    return neg_res, dN, (st[0], st[1], st[2])


def fls_nl_residual2(ctx: Context, nl, Lu: torch.Tensor, u: torch.Tensor, Du: torch.Tensor,
                     f: torch.Tensor, u_prev: Optional[torch.Tensor] = None, stats: bool = True):
    """quasi-linear N(u, Du): returns (neg_res, dN/du, dN/dDu, sums of squares)"""
    n = int(u.numel())
    neg_res, dN, dN2 = torch.empty_like(u), torch.empty_like(u), torch.empty_like(u)
    st = (C.c_double * 3)()
    check(_abi.load().fls_nl_residual2(ctx.handle, C.byref(nl), n, _ptr(Lu), _ptr(u), _ptr(Du),
                                       _ptr(u_prev), _ptr(f), _ptr(neg_res), _ptr(dN), _ptr(dN2),
                                       st if stats else None))
    return neg_res, dN, dN2, (st[0], st[1], st[2])


def fls_axpy(ctx: Context, alpha: float, x: torch.Tensor, y: torch.Tensor,
             out: Optional[torch.Tensor] = None) -> torch.Tensor:
    out = torch.empty_like(y) if out is None else out
    check(_abi.load().fls_axpy(ctx.handle, int(y.numel()), float(alpha), _ptr(x), _ptr(y), _ptr(out)))
    return out


def fls_sample_box(ctx: Context, dim: int, n: int, lo, hi, seed: int, stream: int = 3):
    """Alg. 1 line 2: n seeded uniform points in the box [lo, hi] (device, (n, dim))"""
    X = torch.empty((n, dim), dtype=torch.float64, device=torch.device("cuda", ctx.device))
    lo_h = (C.c_double * dim)(*[float(v) for v in lo])
    hi_h = (C.c_double * dim)(*[float(v) for v in hi])
    check(_abi.load().fls_sample_box(ctx.handle, dim, int(n), lo_h, hi_h,
                                     C.c_uint64(int(seed) & (2**64 - 1)), C.c_uint64(int(stream)),
                                     _ptr(X)))
    return X


def fls_sample_faces(ctx: Context, dim: int, per_face: int, axes: Sequence[int], lo, hi,
                     seed: int, stream: int = 4):
    """per_face points on each face x_k = lo_k, x_k = hi_k for k in axes (device)"""
    mask = 0
    for k in axes:
        mask |= 1 << int(k)
    rows = 2 * per_face * bin(mask).count("1")
    X = torch.empty((rows, dim), dtype=torch.float64, device=torch.device("cuda", ctx.device))
    lo_h = (C.c_double * dim)(*[float(v) for v in lo])
    hi_h = (C.c_double * dim)(*[float(v) for v in hi])
    check(_abi.load().fls_sample_faces(ctx.handle, dim, int(per_face), C.c_uint32(mask), lo_h, hi_h,
                                       C.c_uint64(int(seed) & (2**64 - 1)), C.c_uint64(int(stream)),
                                       _ptr(X)))
    return X


def fls_features_transform(ctx: Context, L, W_hat: torch.Tensor,
                           W: Optional[torch.Tensor] = None) -> torch.Tensor:
    """W_j = L W^_j (App. E reparameterisation); L: host (d, d) array-like"""
    _dev_f64(W_hat, "W_hat")
    F, d = int(W_hat.shape[0]), int(W_hat.shape[1])
    Lh = (C.c_double * (d * d))(*[float(v) for row in L for v in row])
    W = torch.empty_like(W_hat) if W is None else W
    check(_abi.load().fls_features_transform(ctx.handle, d, F, Lh, _ptr(W_hat), _ptr(W)))
    return W


def fls_bandwidth_grad(ctx: Context, W: torch.Tensor, W_hat: torch.Tensor, b: torch.Tensor,
                       blocks, beta: torch.Tensor, normalize: bool = True):
    """dLout/dL (d x d list of lists) for Lout = ||A beta* - b||^2; each block's `values`
    must hold that block's rows of the residual r = A beta* - b"""
    F, d = int(W.shape[0]), int(W.shape[1])
    bs = blocks if isinstance(blocks, BlockSet) else BlockSet(blocks, d)
    G = (C.c_double * (d * d))()
    check(_abi.load().fls_bandwidth_grad(ctx.handle, _ptr(W), _ptr(W_hat), _ptr(b), d, F,
                                         int(bool(normalize)), bs.arr, len(bs.blocks), _ptr(beta), G))
    return [[G[k * d + l] for l in range(d)] for k in range(d)]


class QRFactor:
    """cached Householder factorisation of A (App. I matrix caching):
    factor once, then solve() any number of right-hand sides"""

    def __init__(self, ctx: Context, A: torch.Tensor, n_rows: int, lda: int, n_features: int,
                 sqrt_mu: float = 0.0):
        _dev_f64(A, "A")
        self.ctx = ctx
        self.n_rows, self.n_features = int(n_rows), int(n_features)
        h = C.c_void_p()
        check(_abi.load().fls_qr_factor(ctx.handle, _ptr(A), self.n_rows, int(lda), self.n_features,
                                        float(sqrt_mu), C.byref(h)))
        self.handle = h

    def solve(self, B: torch.Tensor, ldb: Optional[int] = None) -> torch.Tensor:
        """B: (n_rows,) or flat column-major (n_rows x nrhs, ldb); returns (n_features,) or
        (nrhs, n_features) rows = solutions"""
        _dev_f64(B, "B")
        if B.dim() == 1 and ldb is None:
            nrhs, ldb = 1, self.n_rows
        else:
            ldb = self.n_rows if ldb is None else int(ldb)
            nrhs = B.numel() // ldb
        Beta = torch.empty((nrhs, self.n_features), dtype=torch.float64, device=B.device)
        check(_abi.load().fls_qr_solve(self.ctx.handle, self.handle, _ptr(B), ldb, nrhs, _ptr(Beta),
                                       self.n_features))
        return Beta[0] if (B.dim() == 1 and nrhs == 1) else Beta

    def close(self):
        if getattr(self, "handle", None):
            _abi.load().fls_qr_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class BlockSet:
    """marshalled fls_block array (keeps the ctypes structs alive); reusable across calls"""

    def __init__(self, blocks: Sequence[Block], dim: int):
        self.blocks = list(blocks)
        self.ops = []
        self.arr = (_abi.fls_block * len(self.blocks))()
        self.device = None
        for q, blk in enumerate(self.blocks):
            _dev_f64(blk.X, "X")
            if blk.X.dim() != 2 or int(blk.X.shape[1]) != dim:
                raise ValueError(f"block {q}: X must be (n, {dim}), got {tuple(blk.X.shape)}")
            n = int(blk.X.shape[0])
            for t, nm in ((blk.values, "values"), (blk.fields, "fields")):
                if t is not None and t.device != blk.X.device:
                    raise ValueError(f"block {q}: {nm} on {t.device}, X on {blk.X.device}")
            if blk.values is not None and blk.values.numel() != n:
                raise ValueError(f"block {q}: values has {blk.values.numel()} entries for {n} points")
            if blk.fields is not None and (blk.fields.dim() != 2 or int(blk.fields.shape[0]) != n):
                raise ValueError(f"block {q}: fields must be (n={n}, n_fields), got {tuple(blk.fields.shape)}")
            if self.device is None:
                self.device = blk.X.device
            elif blk.X.device != self.device:
                raise ValueError(f"block {q}: X on {blk.X.device}, block 0 on {self.device}")
            op = _Op(dim, blk.terms)
            self.ops.append(op)
            B = self.arr[q]
            B.X = blk.X.data_ptr()
            B.n_points = blk.n
            B.op = C.pointer(op.op)
            if blk.fields is not None:
                _dev_f64(blk.fields, "fields")
                B.coef_fields = blk.fields.data_ptr()
                B.n_fields = int(blk.fields.shape[1])
            else:
                B.coef_fields = None
                B.n_fields = 0
            B.weight = float(blk.weight)
            if blk.values is not None:
                _dev_f64(blk.values, "values")
            B.values = blk.values.data_ptr() if blk.values is not None else None
        self.total = sum(b.n for b in self.blocks)


def fls_assemble(ctx: Context, W: torch.Tensor, b: torch.Tensor, blocks, *,
                 normalize: bool = True, row_begin: int = 0, row_end: Optional[int] = None,
                 A: Optional[torch.Tensor] = None, lda: Optional[int] = None,
                 layout: int = FLS_COL_MAJOR, rhs: Optional[torch.Tensor] = None,
                 with_rhs: bool = True, extra_rows: int = 0):
    """Assemble global rows [row_begin, row_end) of [A | rhs].

    Column-major default: returns (Ab, lda) where Ab is a flat float64 tensor of
    (F + 1) * lda doubles; column j at Ab[j*lda : j*lda + n_local]; rhs in column F.
    extra_rows reserves rows after the local block (e.g. ridge rows for fls_solve).
    Row-major: returns (A (n_local, lda) with lda >= F, rhs (n_local,))."""
    F, dim = _basis(ctx, W, b)
    bs = blocks if isinstance(blocks, BlockSet) else BlockSet(blocks, dim)
    row_end = bs.total if row_end is None else int(row_end)
    n_local = row_end - int(row_begin)
    dev = W.device
    if layout == FLS_COL_MAJOR:
        if lda is None:
            lda = round_up(max(n_local + extra_rows, 1), 4)
        if A is None:
            A = torch.empty(((F + 1) * lda,), dtype=torch.float64, device=dev)
        if with_rhs and rhs is None:
            rhs = A[F * lda:]
    else:
        if lda is None:
            lda = round_up(F, 2)
        if A is None:
            A = torch.empty((max(n_local, 0), lda), dtype=torch.float64, device=dev)
        if with_rhs and rhs is None:
            rhs = torch.empty((max(n_local, 0),), dtype=torch.float64, device=dev)
    _check_outputs(ctx, bs, A, lda, rhs if with_rhs else None, F, n_local, layout)
    check(_abi.load().fls_assemble(ctx.handle, _ptr(W), _ptr(b), dim, F, int(bool(normalize)),
                                   bs.arr, len(bs.blocks), int(row_begin), row_end, _ptr(A),
                                   int(lda), int(layout), _ptr(rhs) if with_rhs else None))
    if layout == FLS_COL_MAJOR:
        return A, lda
    return A, rhs


def _check_outputs(ctx, bs, A, lda, rhs, F, n_local, layout):
    if bs.device is not None and (bs.device.type != "cuda" or bs.device.index != ctx.device):
        raise ValueError(f"the blocks' tensors are on {bs.device}, the ctx on cuda:{ctx.device}")
    _on(ctx, _dev_f64(A, "A"), "A")
    if rhs is not None:
        _on(ctx, _dev_f64(rhs, "rhs"), "rhs")
    # (an lda too small for the layout is the C ABI's FLS_EINVAL, reported by the call)
    lda_ok = int(lda) >= (n_local if layout == FLS_COL_MAJOR else F)
    if n_local > 0 and lda_ok:
        if layout == FLS_COL_MAJOR:
            _need(A, (F - 1) * int(lda) + n_local, "A")
        else:
            _need(A, (n_local - 1) * int(lda) + F, "A")
        if rhs is not None:
            _need(rhs, n_local, "rhs")


def fls_features_assemble(ctx: Context, dim: int, n_features: int, sigma: float, seed: int,
                          blocks, *, W: Optional[torch.Tensor] = None,
                          b: Optional[torch.Tensor] = None, normalize: bool = True,
                          row_begin: int = 0, row_end: Optional[int] = None,
                          A: Optional[torch.Tensor] = None, lda: Optional[int] = None,
                          layout: int = FLS_COL_MAJOR, rhs: Optional[torch.Tensor] = None,
                          extra_rows: int = 0):
    """fls_features + fls_assemble in one call (fused feature draw + prefactor launch).

    Returns (W, b, Ab, lda) column-major or (W, b, A, rhs) row-major."""
    dev = torch.device("cuda", ctx.device)
    F = int(n_features)
    if W is None:
        W = torch.empty((F, dim), dtype=torch.float64, device=dev)
    if b is None:
        b = torch.empty((F,), dtype=torch.float64, device=dev)
    _on(ctx, _dev_f64(W, "W"), "W")
    _on(ctx, _dev_f64(b, "b"), "b")
    _need(W, F * int(dim), "W")
    _need(b, F, "b")
    bs = blocks if isinstance(blocks, BlockSet) else BlockSet(blocks, dim)
    row_end = bs.total if row_end is None else int(row_end)
    n_local = row_end - int(row_begin)
    if layout == FLS_COL_MAJOR:
        if lda is None:
            lda = round_up(max(n_local + extra_rows, 1), 4)
        if A is None:
            A = torch.empty(((F + 1) * lda,), dtype=torch.float64, device=dev)
        if rhs is None:
            rhs = A[F * lda:]
    else:
        if lda is None:
            lda = round_up(F, 2)
        if A is None:
            A = torch.empty((max(n_local, 0), lda), dtype=torch.float64, device=dev)
        if rhs is None:
            rhs = torch.empty((max(n_local, 0),), dtype=torch.float64, device=dev)
    _check_outputs(ctx, bs, A, lda, rhs, F, n_local, layout)
    check(_abi.load().fls_features_assemble(
        ctx.handle, int(dim), F, float(sigma), int(seed) & (2**64 - 1), _ptr(W), _ptr(b),
        int(bool(normalize)), bs.arr, len(bs.blocks), int(row_begin), row_end, _ptr(A), int(lda),
        int(layout), _ptr(rhs)))
    if layout == FLS_COL_MAJOR:
        return W, b, A, lda
    return W, b, A, rhs


def _host_ptr(a):
    if a is None:
        return None
    if isinstance(a, torch.Tensor):
        if a.is_cuda or a.dtype != torch.float64 or not a.is_contiguous():
            raise TypeError("host path needs contiguous float64 CPU tensors / arrays")
        return a.data_ptr()
    if a.dtype.name != "float64" or not a.flags.c_contiguous:
        raise TypeError("host path needs contiguous float64 CPU tensors / arrays")
    return a.ctypes.data


class HostBlockSet:
    """fls_block array over HOST memory (numpy arrays or CPU tensors; pinned is fastest)"""

    def __init__(self, blocks, dim: int):
        self.blocks = list(blocks)
        self.ops = []
        self.arr = (_abi.fls_block * len(self.blocks))()
        for q, blk in enumerate(self.blocks):
            op = _Op(dim, blk.terms)
            self.ops.append(op)
            B = self.arr[q]
            B.X = _host_ptr(blk.X)
            B.n_points = int(blk.X.shape[0])
            B.op = C.pointer(op.op)
            B.coef_fields = _host_ptr(blk.fields) if blk.fields is not None else None
            B.n_fields = int(blk.fields.shape[1]) if blk.fields is not None else 0
            B.weight = float(blk.weight)
            B.values = _host_ptr(blk.values) if blk.values is not None else None
        self.total = sum(int(b.X.shape[0]) for b in self.blocks)


def fls_assemble_host(ctx: Context, W, b, blocks, A, lda: int, rhs=None, *, normalize: bool = True,
                      row_begin: int = 0, row_end: Optional[int] = None, chunk_rows: int = 0):
    """Host-buffer assembly (C ABI fls_assemble_host): W, b, the blocks' arrays, A (flat,
    column-major, >= F * lda doubles) and rhs live in host memory.  Blocking."""
    F, dim = int(W.shape[0]), int(W.shape[1])
    bs = blocks if isinstance(blocks, HostBlockSet) else HostBlockSet(blocks, dim)
    row_end = bs.total if row_end is None else int(row_end)
    check(_abi.load().fls_assemble_host(ctx.handle, _host_ptr(W), _host_ptr(b), dim, F,
                                        int(bool(normalize)), bs.arr, len(bs.blocks),
                                        int(row_begin), row_end, _host_ptr(A), int(lda),
                                        _host_ptr(rhs), int(chunk_rows)))
    return A, rhs


def fls_solve(ctx: Context, Ab: torch.Tensor, n_rows: int, lda: int, n_features: int,
              ridge_rel: float = 0.0, beta: Optional[torch.Tensor] = None):
    """beta = argmin ||A beta - b||^2 + mu ||beta||^2, sqrt(mu) = ridge_rel ||A||_F (reading A16),
    on the column-major [A | b] (destroyed).  With a communicator attached (fls_comm_init*),
    Ab is this rank's rows and the call runs TSQR over the ranks; beta is replicated.
    Returns (beta, residual norm)."""
    _on(ctx, _dev_f64(Ab, "Ab"), "Ab")
    _need(Ab, int(n_features) * int(lda) + int(n_rows), "Ab")
    if beta is None:
        beta = torch.empty((n_features,), dtype=torch.float64, device=Ab.device)
    _need(_on(ctx, _dev_f64(beta, "beta"), "beta"), int(n_features), "beta")
    res = C.c_double(0.0)
    check(_abi.load().fls_solve(ctx.handle, _ptr(Ab), int(n_rows), int(lda), int(n_features),
                                float(ridge_rel), _ptr(beta), C.byref(res)))
    return beta, res.value


def fls_solve_mu(ctx: Context, Ab: torch.Tensor, n_rows: int, lda: int, n_features: int,
                 sqrt_mu: float = 0.0, beta: Optional[torch.Tensor] = None):
    """fls_solve with an ABSOLUTE sqrt(mu) (the Newton step's Tikhonov term)"""
    _on(ctx, _dev_f64(Ab, "Ab"), "Ab")
    _need(Ab, int(n_features) * int(lda) + int(n_rows), "Ab")
    if beta is None:
        beta = torch.empty((n_features,), dtype=torch.float64, device=Ab.device)
    _need(_on(ctx, _dev_f64(beta, "beta"), "beta"), int(n_features), "beta")
    res = C.c_double(0.0)
    check(_abi.load().fls_solve_mu(ctx.handle, _ptr(Ab), int(n_rows), int(lda), int(n_features),
                                   float(sqrt_mu), _ptr(beta), C.byref(res)))
    return beta, res.value


_TRANSPORTS = {"auto": _abi.FLS_TSQR_AUTO, "p2p": _abi.FLS_TSQR_P2P, "nccl": _abi.FLS_TSQR_NCCL}
_TRANSPORT_NAMES = {0: None, _abi.FLS_TSQR_P2P: "p2p", _abi.FLS_TSQR_NCCL: "nccl"}


def fls_comm_unique_id() -> bytes:
    """an NCCL unique id (rank 0 creates it; the caller distributes it to the other ranks)"""
    buf = (C.c_char * _abi.FLS_COMM_ID_BYTES)()
    check(_abi.load().fls_comm_unique_id(buf))
    return bytes(buf)


def fls_comm_init(ctx: Context, uid: bytes, nranks: int, rank: int):
    """attach an NCCL communicator (blocks until every rank has called it)"""
    if len(uid) != _abi.FLS_COMM_ID_BYTES:
        raise ValueError(f"uid must be {_abi.FLS_COMM_ID_BYTES} bytes")
    buf = (C.c_char * _abi.FLS_COMM_ID_BYTES).from_buffer_copy(uid)
    check(_abi.load().fls_comm_init(ctx.handle, buf, int(nranks), int(rank)))


def fls_comm_init_host(ctx: Context, nranks: int, rank: int, allgather):
    """attach a communicator whose control plane is the Python callable
    allgather(data: bytes) -> bytes (nranks * len(data) bytes, rank order); the R factors move
    by peer memory (CUDA IPC)"""
    n = int(nranks)

    def _cb(user, send, recv, nbytes):
        try:
            out = allgather(C.string_at(send, nbytes))
            if len(out) != n * nbytes:
                return 1
            C.memmove(recv, out, len(out))
            return 0
        except Exception:           # a Python error must not unwind through C
            import traceback
            traceback.print_exc()
            return 1

    fn = _abi.HOST_ALLGATHER(_cb)
    coll = _abi.fls_host_coll(None, fn)
    check(_abi.load().fls_comm_init_host(ctx.handle, n, int(rank), C.byref(coll)))
    ctx._comm_keep = (fn, coll, allgather)       # the C side keeps calling fn


def fls_comm_destroy(ctx: Context):
    check(_abi.load().fls_comm_destroy(ctx.handle))
    ctx._comm_keep = None


def fls_comm_config(ctx: Context, transport: str = "auto", force_tsqr: bool = False):
    check(_abi.load().fls_comm_config(ctx.handle, _TRANSPORTS[transport], int(bool(force_tsqr))))


def fls_comm_info(ctx: Context):
    """(nranks, rank, transport of the last solve: None / "p2p" / "nccl")"""
    a, b, c = C.c_int32(), C.c_int32(), C.c_int32()
    check(_abi.load().fls_comm_info(ctx.handle, C.byref(a), C.byref(b), C.byref(c)))
    return a.value, b.value, _TRANSPORT_NAMES.get(c.value, c.value)


def fls_solve_stacked(ctx: Context, S: torch.Tensor, n_blocks: int, kb: int, lds: int,
                      n_features: int, sqrt_mu: float = 0.0, beta: Optional[torch.Tensor] = None):
    """TSQR root step: beta of the stacked triangular factors [R_r | c_r] (block r at rows
    [r kb, (r+1) kb) of the flat column-major S), structure-exploiting; S is not modified."""
    _dev_f64(S, "S")
    if beta is None:
        beta = torch.empty((n_features,), dtype=torch.float64, device=S.device)
    res = C.c_double(0.0)
    check(_abi.load().fls_solve_stacked(ctx.handle, _ptr(S), int(n_blocks), int(kb), int(lds),
                                        int(n_features), float(sqrt_mu), _ptr(beta), C.byref(res)))
    return beta, res.value


def fls_geqrf(ctx: Context, M: torch.Tensor, n_rows: int, lda: int, n_cols: int,
              tau: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Householder QR of the flat column-major block M in place (geqrf format); returns tau"""
    _dev_f64(M, "M")
    if M.numel() < lda * (n_cols - 1) + n_rows:
        raise ValueError("M too small for n_rows x n_cols at lda")
    k = min(n_rows, n_cols)
    tau = torch.empty((k,), dtype=torch.float64, device=M.device) if tau is None else tau
    check(_abi.load().fls_geqrf(ctx.handle, _ptr(M), int(n_rows), int(lda), int(n_cols), _ptr(tau)))
    return tau


def fls_qr_r(ctx: Context, M: torch.Tensor, n_rows: int, lda: int, n_cols: int,
             R: Optional[torch.Tensor] = None, ldr: Optional[int] = None, R_ptr: Optional[int] = None):
    """local Householder QR, R (upper trapezoid) into R -- or into raw device memory R_ptr (e.g.
    a peer process's buffer mapped by fls_ipc_open: the copy kernel's stores are the transfer)"""
    k = min(n_rows, n_cols)
    ldr = k if ldr is None else ldr
    if R_ptr is None and R is None:
        R = torch.empty((n_cols * ldr,), dtype=torch.float64, device=M.device)
    dst = C.c_void_p(R_ptr) if R_ptr is not None else _ptr(R)
    check(_abi.load().fls_qr_r(ctx.handle, _ptr(M), int(n_rows), int(lda), int(n_cols), dst,
                               int(ldr)))
    return R, ldr


def fls_ipc_handle(ctx: Context, t: torch.Tensor):
    """(CUDA IPC handle of the allocation holding device tensor t, byte offset of t in it)"""
    buf = (C.c_char * _abi.FLS_IPC_HANDLE_BYTES)()
    off = C.c_int64(0)
    check(_abi.load().fls_ipc_handle(ctx.handle, C.c_void_p(t.data_ptr()), buf, C.byref(off)))
    return bytes(buf), int(off.value)


def fls_ipc_open(ctx: Context, handle: bytes) -> int:
    """map another process's exported allocation; returns its base device address here"""
    buf = (C.c_char * _abi.FLS_IPC_HANDLE_BYTES).from_buffer_copy(handle)
    out = C.c_void_p()
    check(_abi.load().fls_ipc_open(ctx.handle, buf, C.byref(out)))
    return int(out.value)


def fls_ipc_close(ctx: Context, ptr: int):
    check(_abi.load().fls_ipc_close(ctx.handle, C.c_void_p(ptr)))


def fls_frob2(ctx: Context, A: torch.Tensor, n_rows: int, lda: int, n_cols: int) -> float:
    _on(ctx, _dev_f64(A, "A"), "A")
    if n_rows > 0 and n_cols > 0:
        _need(A, (int(n_cols) - 1) * int(lda) + int(n_rows), "A")
    out = C.c_double(0.0)
    check(_abi.load().fls_frob2(ctx.handle, _ptr(A), int(n_rows), int(lda), int(n_cols),
                                C.byref(out)))
    return out.value


def fls_eval_block(ctx: Context, W: torch.Tensor, b: torch.Tensor, beta: torch.Tensor, block: Block,
                   normalize: bool = True, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """A_block @ beta for one row block (its operator, coefficient fields and weight), without
    materialising A"""
    F, dim = _basis(ctx, W, b)
    _need(_on(ctx, _dev_f64(beta, "beta"), "beta"), F, "beta")
    bs = BlockSet([block], dim)
    _on(ctx, block.X, "block.X")
    if out is None:
        out = torch.empty((block.n,), dtype=torch.float64, device=W.device)
    _need(_on(ctx, _dev_f64(out, "out"), "out"), block.n, "out")
    check(_abi.load().fls_eval_block(ctx.handle, _ptr(W), _ptr(b), dim, F, int(bool(normalize)),
                                     _ptr(beta), bs.arr, _ptr(out)))
    return out


def fls_eval(ctx: Context, W: torch.Tensor, b: torch.Tensor, beta: torch.Tensor, X: torch.Tensor,
             terms: Optional[Sequence[Term]] = None, normalize: bool = True,
             out: Optional[torch.Tensor] = None) -> torch.Tensor:
    F, dim = _basis(ctx, W, b)
    for t, nm in ((beta, "beta"), (X, "X")):
        _on(ctx, _dev_f64(t, nm), nm)
    _need(beta, F, "beta")
    if X.dim() != 2 or int(X.shape[1]) != dim:
        raise ValueError(f"X must be (n, {dim}), got {tuple(X.shape)}")
    n = int(X.shape[0])
    if out is None:
        out = torch.empty((n,), dtype=torch.float64, device=X.device)
    _need(_on(ctx, _dev_f64(out, "out"), "out"), n, "out")
    op = _Op(dim, terms) if terms is not None else None
    check(_abi.load().fls_eval(ctx.handle, _ptr(W), _ptr(b), dim, F, int(bool(normalize)),
                               _ptr(beta), C.pointer(op.op) if op else None, _ptr(X), n, _ptr(out)))
    return out
