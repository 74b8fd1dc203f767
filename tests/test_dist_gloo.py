"""Multi-rank host logic on CPU (world_size 2-3, gloo): row sharding, dist.py's attachment of
the libfls communicator (unique-id broadcast, host-callback allgather) and the TSQR combine,
with test-double arithmetic (numpy QR / triangular solve) in place of the libfls GPU calls.
The GPU arithmetic itself is covered by the -m gpu tests."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from scipy.linalg import solve_triangular

from paper_2602_10541_b200.dist import shard_range, tsqr_solve


class NumpyOps:
    """CPU stand-ins with the exact libfls calling conventions (column-major, flat buffers)"""

    def frob2(self, Ab, n_rows, lda, F):
        M = Ab[: F * lda].view(F, lda)[:, :n_rows].numpy()
        return float((M * M).sum())

    def qr_r(self, Ab, n_rows, lda, ncols):
        M = Ab[: ncols * lda].view(ncols, lda)[:, :n_rows].numpy().T      # (n_rows, ncols)
        R = np.linalg.qr(M, mode="r")                                       # (k, ncols)
        k = R.shape[0]
        return torch.from_numpy(np.ascontiguousarray(R.T).ravel()), k

    def solve(self, M, n_rows, lda, F, sqrt_mu):
        Mv = M[: (F + 1) * lda].view(F + 1, lda)[:, :n_rows].numpy().T     # (n_rows, F+1)
        if sqrt_mu > 0:
            Mv = np.vstack([Mv, np.hstack([sqrt_mu * np.eye(F), np.zeros((F, 1))])])
        R = np.linalg.qr(Mv, mode="r")
        beta = solve_triangular(R[:F, :F], R[:F, F])
        res = abs(R[F, F]) if R.shape[0] > F else 0.0
        return torch.from_numpy(beta), float(res)

    def solve_stacked(self, S, n_blocks, kb, lds, F, sqrt_mu):
        # the stack in block order is a plain [A | b] of n_blocks * kb rows
        M = torch.zeros((F + 1) * (n_blocks * kb + F), dtype=torch.float64)
        ld = n_blocks * kb + F
        M.view(F + 1, ld)[:, :n_blocks * kb] = S[: (F + 1) * lds].view(F + 1, lds)[:, :n_blocks * kb]
        return self.solve(M, n_blocks * kb, ld, F, sqrt_mu)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class FakeComm:
    """CPU stand-in for libfls's communicator with its control-plane protocol: fls_solve on a
    ctx with a host-callback comm exchanges, through the caller's allgather, a fixed-size header
    per rank (rows k_r, ||A_r||_F^2) and then each rank's R factor zero-padded to kmax rows; the
    stacked factors are solved with the ridge rows (sqrt(mu) = tau sqrt(sum_r ||A_r||_F^2)).
    What it tests here: dist.py's wiring -- the unique-id broadcast, the allgather callable
    (rank order, byte counts) and the replicated result."""

    def __init__(self):
        self.uid = None
        self.ag = None

    def unique_id(self):
        return bytes(np.random.default_rng().integers(0, 256, 128, dtype=np.uint8))

    def init_nccl(self, ctx, uid, nranks, rank):
        self.uid, self.nranks, self.rank = uid, nranks, rank

    def init_host(self, ctx, nranks, rank, allgather):
        self.ag, self.nranks, self.rank = allgather, nranks, rank

    def config(self, ctx, transport, force):
        self.cfg = (transport, force)

    def info(self, ctx):
        return self.nranks, self.rank, "p2p"

    def solve(self, ctx, Ab, n, lda, F, ridge_rel):
        nc = F + 1
        M = Ab[: nc * lda].view(nc, lda)[:, :n].numpy().T            # (n, F+1)
        hdr = np.array([min(n, nc), float((M[:, :F] ** 2).sum())])
        allh = np.frombuffer(self.ag(hdr.tobytes()), dtype=np.float64).reshape(self.nranks, 2)
        kmax = int(allh[:, 0].max())
        R = np.linalg.qr(M, mode="r") if n > 0 else np.zeros((0, nc))
        pad = np.zeros((kmax, nc))
        pad[: R.shape[0]] = R
        stack = np.frombuffer(self.ag(pad.tobytes()), dtype=np.float64).reshape(self.nranks * kmax, nc)
        sq = ridge_rel * np.sqrt(allh[:, 1].sum())            # rank-order sum
        if sq > 0:
            stack = np.vstack([stack, np.hstack([sq * np.eye(F), np.zeros((F, 1))])])
        Rs = np.linalg.qr(stack, mode="r")
        beta = solve_triangular(Rs[:F, :F], Rs[:F, F])
        return torch.from_numpy(beta), float(abs(Rs[F, F]))


def _worker(rank, world, port, case, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_10541_b200 import dist as fdist
        R, F, ridge = case
        g = np.random.default_rng(42)
        A = g.normal(size=(R, F))
        b = g.normal(size=R)
        a, e = shard_range(R, rank, world)
        n = e - a
        lda = max(4, ((n + 3) // 4) * 4)
        Ab = torch.zeros((F + 1) * lda, dtype=torch.float64)
        V = Ab.view(F + 1, lda)
        V[:F, :n] = torch.from_numpy(A[a:e].T.copy())
        V[F, :n] = torch.from_numpy(b[a:e].copy())

        class Ctx:
            pass
        fake = FakeComm()
        beta, _ = tsqr_solve(Ab, n, lda, F, ridge_rel=ridge, ctx=Ctx(), ops=fake)
        out[rank] = (beta.numpy().tolist(), fdist.LAST_TRANSPORT, fake.ag is not None)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [(2, (300, 40, 0.0)), (2, (50, 40, 0.0)), (2, (60, 40, 1e-3)),
                                        (2, (7, 10, 0.5)), (3, (5, 10, 0.5))])
def test_tsqr_ranks_match_single_lstsq(world, case):
    """gloo group -> host-callback control plane; ranks with fewer rows than features (7 rows
    over 2 ranks, 5 over 3) give trapezoidal factors"""
    R, F, ridge = case
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), case, out), nprocs=world, join=True)
    g = np.random.default_rng(42)
    A = g.normal(size=(R, F))
    b = g.normal(size=R)
    if ridge > 0:
        sq = ridge * np.linalg.norm(A)
        A2 = np.vstack([A, sq * np.eye(F)])
        b2 = np.concatenate([b, np.zeros(F)])
    else:
        A2, b2 = A, b
    ref, *_ = np.linalg.lstsq(A2, b2, rcond=None)
    for r in range(world):
        got, used, host = out[r]
        assert host and used == "p2p"
        assert np.allclose(got, ref, rtol=1e-9, atol=1e-9 * np.abs(ref).max())
    assert all(out[r][0] == out[0][0] for r in range(world))


def _worker_uid(rank, world, port, out):
    """NCCL control plane wiring: rank 0 of the (sub)group makes the id, every member gets the
    same bytes; a subgroup that does not start at global rank 0 maps its root correctly"""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_10541_b200.dist import attach_comm

        class Ctx:
            pass
        sub = dist.new_group([1, 2])
        fake = FakeComm()
        if rank in (1, 2):
            used = attach_comm(Ctx(), sub, control="nccl", ops=fake)
            out[rank] = (fake.uid, fake.nranks, fake.rank, used)
        fake0 = FakeComm()
        used0 = attach_comm(Ctx(), None, control="nccl", transport="nccl", ops=fake0)
        out[10 + rank] = (fake0.uid, fake0.nranks, fake0.rank, used0, fake0.cfg)
    finally:
        dist.destroy_process_group()


def test_nccl_unique_id_broadcast_and_subgroup_root():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_uid, args=(3, _free_port(), out), nprocs=3, join=True)
    assert out[1][0] == out[2][0] and len(out[1][0]) == 128
    assert (out[1][1], out[1][2], out[2][2]) == (2, 0, 1) and out[1][3] == "nccl"
    assert out[10][0] == out[11][0] == out[12][0] != out[1][0]
    assert [out[10 + r][2] for r in range(3)] == [0, 1, 2]
    assert out[10][4] == ("nccl", False)


def _worker_allgather(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_10541_b200.dist import host_allgather
        ag = host_allgather()
        out[rank] = ag(bytes([rank, 2 * rank, 255]) * 5)
    finally:
        dist.destroy_process_group()


def test_host_allgather_rank_order_and_length():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_allgather, args=(3, _free_port(), out), nprocs=3, join=True)
    want = b"".join(bytes([r, 2 * r, 255]) * 5 for r in range(3))
    assert all(out[r] == want for r in range(3))


@pytest.mark.parametrize("P,R,F,ridge", [(4, 300, 40, 0.0), (8, 100, 40, 0.0), (3, 30, 20, 0.1)])
def test_tsqr_local_logical_blocks(P, R, F, ridge):
    """single-process TSQR over P logical row blocks (the 1-GPU mode) == one lstsq"""
    from paper_2602_10541_b200.dist import tsqr_local
    g = np.random.default_rng(P)
    A = g.normal(size=(R, F))
    b = g.normal(size=R)
    blocks = []
    for r in range(P):
        a, e = shard_range(R, r, P)
        n = e - a
        lda = max(4, ((n + 3) // 4) * 4)
        Ab = torch.zeros((F + 1) * lda, dtype=torch.float64)
        V = Ab.view(F + 1, lda)
        V[:F, :n] = torch.from_numpy(A[a:e].T.copy())
        V[F, :n] = torch.from_numpy(b[a:e].copy())
        blocks.append((Ab, n, lda))
    beta, _ = tsqr_local(blocks, F, ridge_rel=ridge, ops=NumpyOps())
    if ridge > 0:
        sq = ridge * np.linalg.norm(A)
        A, b = np.vstack([A, sq * np.eye(F)]), np.concatenate([b, np.zeros(F)])
    ref, *_ = np.linalg.lstsq(A, b, rcond=None)
    assert np.allclose(beta.numpy(), ref, rtol=1e-9, atol=1e-9 * np.abs(ref).max())


def test_shard_ranges_partition_rows():
    for R in (0, 1, 7, 1002, 2_097_152):
        for P in (1, 2, 3, 4, 8):
            spans = [shard_range(R, r, P) for r in range(P)]
            assert spans[0][0] == 0 and spans[-1][1] == R
            assert all(spans[i][1] == spans[i + 1][0] for i in range(P - 1))
            sizes = [e - a for a, e in spans]
            assert max(sizes) - min(sizes) <= 1
