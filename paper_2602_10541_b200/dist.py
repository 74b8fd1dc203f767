"""Multi-GPU plumbing: row sharding of the stacked system and the attachment of libfls's
communicator for the TSQR least-squares solve.

Assembly needs no collective: rank r owns global rows
[floor(r R / P), floor((r+1) R / P)) and every rank regenerates W, b from the seed.
The solve has one real exchange step (TSQR, "QR or SVD"; Tikhonov form P:L158), and it
runs INSIDE libfls (csrc/fls_comm.cu): fls_solve on a ctx with a communicator does the local QR,
moves the R factors to the root (peer-memory stores over CUDA IPC, or NCCL send/recv), solves
the stacked factors there and replicates beta on every rank.  This module only
  - creates that communicator from a torch.distributed group: an NCCL communicator (the
    ncclUniqueId made by libfls on rank 0, broadcast through the group) when the group is NCCL
    on CUDA, else the host-callback control plane (fls_comm_init_host) over the group's
    all_gather -- which also serves several processes sharing one GPU (NCCL refuses that);
  - calls fls_solve.
The comm calls are injectable (`ops`) so the wiring can be tested on CPU with gloo
(tests/test_dist_gloo.py); the arithmetic is covered by the -m gpu tests.
"""
from __future__ import annotations

import math
from typing import Callable, Optional, Tuple

import torch
import torch.distributed as dist


LAST_TRANSPORT = None   # transport the last multi-rank tsqr_solve used ("p2p" / "nccl")


def shard_range(n_rows: int, rank: int, world: int) -> Tuple[int, int]:
    return (rank * n_rows) // world, ((rank + 1) * n_rows) // world


class _FlsComm:
    """default: libfls's communicator calls"""

    def __init__(self):
        from . import fls
        self.fls = fls

    def unique_id(self) -> bytes:
        return self.fls.fls_comm_unique_id()

    def init_nccl(self, ctx, uid, nranks, rank):
        self.fls.fls_comm_init(ctx, uid, nranks, rank)

    def init_host(self, ctx, nranks, rank, allgather):
        self.fls.fls_comm_init_host(ctx, nranks, rank, allgather)

    def config(self, ctx, transport, force_tsqr):
        self.fls.fls_comm_config(ctx, transport, force_tsqr)

    def info(self, ctx):
        return self.fls.fls_comm_info(ctx)

    def solve(self, ctx, Ab, n_local, lda, F, ridge_rel):
        return self.fls.fls_solve(ctx, Ab, n_local, lda, F, ridge_rel)


def host_allgather(group=None) -> Callable[[bytes], bytes]:
    """allgather of equal-length byte strings over a torch.distributed group, rank order (the
    control plane libfls calls back into during fls_solve)"""

    def allgather(data: bytes) -> bytes:
        world = dist.get_world_size(group)
        if dist.get_backend(group) == "nccl":
            dev = torch.device("cuda", torch.cuda.current_device())
        else:
            dev = torch.device("cpu")
        t = torch.frombuffer(bytearray(data), dtype=torch.uint8).to(dev) if data else \
            torch.empty(0, dtype=torch.uint8, device=dev)
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t, group=group)
        return b"".join(o.cpu().numpy().tobytes() for o in out)

    return allgather


def _group_root(group) -> int:
    """global rank of the group's rank 0 (broadcast_object_list takes a global src)"""
    return 0 if group is None else dist.get_global_rank(group, 0)


def attach_comm(ctx, group=None, *, control: str = "auto", transport: str = "auto",
                force_tsqr: bool = False, ops=None) -> Optional[str]:
    """attach a libfls communicator for `group` to ctx (once).  control: "nccl" (NCCL
    communicator; one rank per GPU), "host" (callbacks over the group), "auto" = nccl for NCCL
    groups on CUDA, else host.  Returns the control plane used (None: single process, no
    group)."""
    ops = ops if ops is not None else _FlsComm()
    if getattr(ctx, "_fls_comm_control", None):
        return ctx._fls_comm_control
    if not dist.is_initialized():
        return None
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if control == "auto":
        control = "nccl" if dist.get_backend(group) == "nccl" else "host"
    if control == "nccl":
        obj = [ops.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=_group_root(group), group=group)
        ops.init_nccl(ctx, obj[0], world, rank)
    else:
        ops.init_host(ctx, world, rank, host_allgather(group))
    if transport != "auto" or force_tsqr:
        ops.config(ctx, transport, force_tsqr)
    ctx._fls_comm_control = control
    return control


def tsqr_solve(Ab: torch.Tensor, n_local: int, lda: int, F: int, *, ridge_rel: float = 0.0,
               ctx=None, group=None, control: str = "auto", transport: str = "auto",
               ops=None) -> Tuple[torch.Tensor, float]:
    """beta = argmin ||A beta - b||^2 + mu ||beta||^2 (sqrt(mu) = ridge_rel ||A||_F over all
    ranks) for [A | b] row-sharded over the group: this rank's column-major [A_r | b_r] (flat,
    (F+1) * lda, destroyed).  Returns (beta replicated on every rank, residual norm)."""
    global LAST_TRANSPORT
    ops = ops if ops is not None else _FlsComm()
    attach_comm(ctx, group, control=control, transport=transport, ops=ops)
    beta, res = ops.solve(ctx, Ab, n_local, lda, F, ridge_rel)
    if getattr(ctx, "_fls_comm_control", None):
        LAST_TRANSPORT = ops.info(ctx)[2]
    return beta, res


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


class _FlsLocalOps:
    def __init__(self, ctx):
        from . import fls
        self.fls = fls
        self.ctx = ctx

    def frob2(self, Ab, n_rows, lda, F):
        return self.fls.fls_frob2(self.ctx, Ab, n_rows, lda, F)

    def qr_r(self, Ab, n_rows, lda, ncols):
        return self.fls.fls_qr_r(self.ctx, Ab, n_rows, lda, ncols)

    def solve_stacked(self, S, n_blocks, kb, lds, F, sqrt_mu):
        return self.fls.fls_solve_stacked(self.ctx, S, n_blocks, kb, lds, F, sqrt_mu)


def tsqr_local(blocks, F: int, *, ridge_rel: float = 0.0, ctx=None, ops=None):
    """TSQR over P row blocks held by ONE process (the 1-GPU test mode of SURVEY §4.5):
    blocks = [(Ab_r, n_r, lda_r)], each a column-major [A_r | b_r] (destroyed)."""
    ops = ops if ops is not None else _FlsLocalOps(ctx)
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
