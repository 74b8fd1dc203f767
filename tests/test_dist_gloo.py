"""Multi-rank host logic on CPU (world_size 2, gloo): row sharding and the TSQR combine of
paper_2602_10541_b200.dist, with test-double arithmetic (numpy QR / triangular solve) in place
of the libfls GPU calls.  The GPU arithmetic itself is covered by the -m gpu tests."""
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


class NoIpcOps(NumpyOps):
    """the root cannot export its buffer (e.g. VMM allocations): every rank must fall back"""

    def ipc_handle(self, t):
        raise RuntimeError("no CUDA IPC here")


def _worker_p2p_fallback(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_10541_b200 import dist as fdist
        R, F = 120, 16
        g = np.random.default_rng(7)
        A = g.normal(size=(R, F))
        b = g.normal(size=R)
        a, e = shard_range(R, rank, world)
        n = e - a
        lda = ((n + 3) // 4) * 4
        Ab = torch.zeros((F + 1) * lda, dtype=torch.float64)
        V = Ab.view(F + 1, lda)
        V[:F, :n] = torch.from_numpy(A[a:e].T.copy())
        V[F, :n] = torch.from_numpy(b[a:e].copy())
        beta, _ = tsqr_solve(Ab, n, lda, F, ops=NoIpcOps(), transport="p2p")
        out[rank] = (beta.numpy().tolist(), fdist.LAST_TRANSPORT)
    finally:
        dist.destroy_process_group()


def test_tsqr_p2p_falls_back_to_collective_on_every_rank():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_p2p_fallback, args=(2, _free_port(), out), nprocs=2, join=True)
    g = np.random.default_rng(7)
    A = g.normal(size=(120, 16))
    b = g.normal(size=120)
    ref, *_ = np.linalg.lstsq(A, b, rcond=None)
    for r in range(2):
        beta, used = out[r]
        assert used == "collective"
        assert np.allclose(beta, ref, rtol=1e-9, atol=1e-9 * np.abs(ref).max())


def _worker(rank, world, port, case, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
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
        beta, _ = tsqr_solve(Ab, n, lda, F, ridge_rel=ridge, ops=NumpyOps())
        out[rank] = beta.numpy().tolist()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [(300, 40, 0.0), (50, 40, 0.0), (60, 40, 1e-3), (7, 10, 0.5)])
def test_tsqr_two_ranks_matches_single_lstsq(case):
    R, F, ridge = case
    mgr = mp.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(2, port, case, out), nprocs=2, join=True)
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
    for r in range(2):
        got = np.array(out[r])
        assert np.allclose(got, ref, rtol=1e-9, atol=1e-9 * np.abs(ref).max())
    assert out[0] == out[1]          # replicated bit-identically (broadcast)


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
