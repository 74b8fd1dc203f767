"""Multi-GPU plumbing: row sharding of the stacked system and the TSQR least-squares solve.

Assembly needs no collective: rank r owns global rows
[floor(r R / P), floor((r+1) R / P)) and every rank regenerates W, b from the seed.
The solve has one real exchange step (TSQR, "QR or SVD"; Tikhonov form P:L158):

    local:  [A_r | b_r] = Q_r R_r                      (fls_qr_r, Householder QR on each GPU)
    gather: R_0 .. R_{P-1} -> root   (default on GPUs: each rank's R-extraction kernel stores
                                      straight into the root's buffer over CUDA IPC peer
                                      memory; else a torch.distributed gather)
    root:   [R_0; ...; R_{P-1}; sqrt(mu) I | 0] = Q R   (fls_solve_stacked: the triangles' zeros
                                                     skipped, blocked QR + trsv)
    bcast:  beta

`ridge_rel` = tau of DESIGN.md reading A16: sqrt(mu) = tau ||A||_F with ||A||_F^2 summed over
ranks (all_reduce).  Every arithmetic step runs in libfls / cuSOLVER; this module only moves
tensors.  The local-QR / solve / norm callables are injectable so the host-side combine logic
can be tested on CPU with gloo (tests/test_dist_gloo.py).
"""
from __future__ import annotations

import math
import os
from typing import Callable, Optional, Tuple

import torch
import torch.distributed as dist


LAST_TRANSPORT = None   # transport the last multi-rank tsqr_solve used ("p2p" / "collective")


def shard_range(n_rows: int, rank: int, world: int) -> Tuple[int, int]:
    return (rank * n_rows) // world, ((rank + 1) * n_rows) // world


class _FlsOps:
    """default arithmetic: libfls on the current device"""

    def __init__(self, ctx):
        from . import fls
        self.fls = fls
        self.ctx = ctx

    def frob2(self, Ab, n_rows, lda, F):
        return self.fls.fls_frob2(self.ctx, Ab, n_rows, lda, F)

    def qr_r(self, Ab, n_rows, lda, ncols):
        R, ldr = self.fls.fls_qr_r(self.ctx, Ab, n_rows, lda, ncols)
        return R, ldr

    def solve(self, M, n_rows, lda, F, sqrt_mu):
        return self.fls.fls_solve(self.ctx, M, n_rows, lda, F, sqrt_mu)

    def solve_stacked(self, S, n_blocks, kb, lds, F, sqrt_mu):
        return self.fls.fls_solve_stacked(self.ctx, S, n_blocks, kb, lds, F, sqrt_mu)

    # peer-memory transport (CUDA IPC over NVLink / NVSwitch)
    def qr_r_into(self, Ab, n_rows, lda, ncols, dst_ptr, ldr):
        self.fls.fls_qr_r(self.ctx, Ab, n_rows, lda, ncols, ldr=ldr, R_ptr=dst_ptr)

    def ipc_handle(self, t):
        return self.fls.fls_ipc_handle(self.ctx, t)

    def ipc_open(self, handle):
        return self.fls.fls_ipc_open(self.ctx, handle)

    def ipc_close(self, ptr):
        self.fls.fls_ipc_close(self.ctx, ptr)


def _combine(ops, Rs, ks, F, sqrt_mu, dev):
    """root step of TSQR: stack the (F+1) x k_r upper-trapezoidal factors in blocks of kmax rows
    and solve the stack with its ridge rows (fls_solve_stacked exploits the triangles)"""
    nc = F + 1
    kmax = max(ks)
    P = len(Rs)
    lds = ((P * kmax + 3) // 4) * 4
    S = torch.zeros((nc * lds,), dtype=torch.float64, device=dev)
    Sv = S.view(nc, lds)
    for r, (R, k) in enumerate(zip(Rs, ks)):
        Sv[:, r * kmax:r * kmax + k] = R[:, :k]
    return ops.solve_stacked(S, P, kmax, lds, F, sqrt_mu)


def tsqr_local(blocks, F: int, *, ridge_rel: float = 0.0, ctx=None, ops=None):
    """TSQR over P row blocks held by ONE process (the 1-GPU test mode of SURVEY §4.5):
    blocks = [(Ab_r, n_r, lda_r)], each a column-major [A_r | b_r] (destroyed)."""
    ops = ops if ops is not None else _FlsOps(ctx)
    dev = blocks[0][0].device
    nc = F + 1
    sqrt_mu = 0.0
    if ridge_rel > 0.0:
        fro2 = sum(ops.frob2(Ab, n, lda, F) for Ab, n, lda in blocks if n > 0)
        sqrt_mu = ridge_rel * math.sqrt(fro2)
    Rs, ks = [], []
    for Ab, n, lda in blocks:
        k = min(n, nc)
        if k == 0:
            continue
        R, ldr = ops.qr_r(Ab, n, lda, nc)
        Rs.append(R[: nc * ldr].view(nc, ldr))
        ks.append(k)
    return _combine(ops, Rs, ks, F, sqrt_mu, dev)


def _tsqr_p2p(ops, Ab, n_local, lda, F, sqrt_mu, group, root, world, rank, dev, cdev):
    """TSQR exchange over peer memory: the root allocates the stacking buffer S (rank r's R
    factor at rows [r kmax, r kmax + k_r), zero rows elsewhere, ridge rows after), exports it
    by CUDA IPC, and every rank's fls_qr_r writes its R straight into S (the copy kernel's
    remote stores over NVLink are the transfer).  Host barrier, then the root solves."""
    nc = F + 1
    k = min(n_local, nc)
    ks = torch.tensor([k], dtype=torch.int64, device=cdev)
    all_k = [torch.zeros_like(ks) for _ in range(world)]
    dist.all_gather(all_k, ks, group=group)
    kmax = max(int(t.item()) for t in all_k)
    K = world * kmax
    ldm = ((K + 3) // 4) * 4
    S = None
    obj = [None]
    if rank == root:
        S = torch.zeros((nc * ldm,), dtype=torch.float64, device=dev)
        if dev.type == "cuda":
            torch.cuda.synchronize(dev)
        try:
            obj = [ops.ipc_handle(S)]
        except Exception:        # e.g. an allocator whose memory cannot be exported (VMM)
            obj = [None]
    dist.broadcast_object_list(obj, src=root, group=group)
    if obj[0] is None:           # every rank falls back to the collective transport
        return None
    handle, off = obj[0]
    base, ok = None, 1
    try:
        base = S.data_ptr() if rank == root else ops.ipc_open(handle) + off
    except Exception:            # e.g. no peer access between these GPUs
        ok = 0
    flag = torch.tensor([ok], dtype=torch.int64, device=cdev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    if int(flag.item()) == 0:    # every rank falls back to the collective transport
        if base is not None and rank != root:
            ops.ipc_close(base - off)
        return None
    try:
        if k > 0:
            ops.qr_r_into(Ab, n_local, lda, nc, base + 8 * rank * kmax, ldm)   # blocking
        dist.barrier(group=group)
    finally:
        if rank != root:
            ops.ipc_close(base - off)
    beta = torch.empty((F,), dtype=torch.float64, device=cdev)
    res = 0.0
    if rank == root:
        b_root, res = ops.solve_stacked(S, world, kmax, ldm, F, sqrt_mu)
        beta.copy_(b_root)
    dist.broadcast(beta, src=root, group=group)
    return beta.to(dev), res


def tsqr_solve(Ab: torch.Tensor, n_local: int, lda: int, F: int, *, ridge_rel: float = 0.0,
               ctx=None, ops=None, group=None, root: int = 0,
               transport: str = "auto") -> Tuple[torch.Tensor, float]:
    """beta = argmin ||A beta - b||^2 + mu ||beta||^2 for [A | b] row-sharded over the ranks.

    Ab: this rank's column-major [A_r | b_r] (flat, (F+1) * lda, destroyed).
    transport: "p2p" (R factors written into the root's buffer over CUDA IPC peer memory),
    "collective" (gather through torch.distributed), "auto" = p2p for NCCL process groups on
    CUDA unless FLS_TSQR_TRANSPORT=collective.
    Returns (beta replicated on every rank, residual norm on root / 0.0 elsewhere)."""
    ops = ops if ops is not None else _FlsOps(ctx)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    dev = Ab.device
    # collectives run on the device for NCCL; gloo (CPU tests, or FLS_DIST_BACKEND=gloo to
    # exercise the multi-rank host logic on one GPU) exchanges host copies
    cdev = torch.device("cpu") if (world > 1 and dist.get_backend(group) == "gloo") else dev
    nc = F + 1
    sqrt_mu = 0.0
    if ridge_rel > 0.0:
        fro2 = torch.tensor([ops.frob2(Ab, n_local, lda, F) if n_local > 0 else 0.0],
                            dtype=torch.float64, device=cdev)
        if world > 1:
            dist.all_reduce(fro2, op=dist.ReduceOp.SUM, group=group)
        sqrt_mu = ridge_rel * math.sqrt(float(fro2.item()))
    if world == 1:
        if ridge_rel > 0.0 and lda < n_local + F:
            raise ValueError("ridge needs lda >= n_local + F (reserve extra_rows=F)")
        beta, res = ops.solve(Ab, n_local, lda, F, sqrt_mu)
        return beta, res

    if transport == "auto":
        transport = os.environ.get("FLS_TSQR_TRANSPORT", "")
        if transport not in ("p2p", "collective"):
            transport = "p2p" if (dev.type == "cuda" and dist.get_backend(group) == "nccl") else "collective"
    global LAST_TRANSPORT
    if transport == "p2p":
        out = _tsqr_p2p(ops, Ab, n_local, lda, F, sqrt_mu, group, root, world, rank, dev, cdev)
        if out is not None:
            LAST_TRANSPORT = "p2p"
            return out
    LAST_TRANSPORT = "collective"

    # collective transport: local R factor, padded to kmax rows (zero rows change nothing)
    k = min(n_local, nc)
    if k > 0:
        R, ldr = ops.qr_r(Ab, n_local, lda, nc)
        Rl = R[: nc * ldr].view(nc, ldr)[:, :k]           # (nc, k): column j = R[0:k, j]
    else:
        Rl = torch.zeros((nc, 0), dtype=torch.float64, device=dev)
    ks = torch.tensor([k], dtype=torch.int64, device=cdev)
    all_k = [torch.zeros_like(ks) for _ in range(world)]
    dist.all_gather(all_k, ks, group=group)
    all_k = [int(t.item()) for t in all_k]
    kmax = max(all_k)
    send = torch.zeros((nc, kmax), dtype=torch.float64, device=cdev)
    send[:, :k] = Rl.to(cdev)
    gathered = [torch.empty_like(send) for _ in range(world)] if rank == root else None
    dist.gather(send, gathered, dst=root, group=group)
    beta = torch.empty((F,), dtype=torch.float64, device=cdev)
    res = 0.0
    if rank == root:
        b_root, res = _combine(ops, [g.to(dev) for g in gathered], all_k, F, sqrt_mu, dev)
        beta.copy_(b_root)
    dist.broadcast(beta, src=root, group=group)
    return beta.to(dev), res
