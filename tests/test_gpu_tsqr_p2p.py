"""TSQR with the peer-memory transport (CUDA IPC): two processes on the one available GPU, host
(gloo) synchronisation only -- no kernel waits on another process's kernel.  Rank 1's
R-extraction kernel stores straight into rank 0's stacking buffer; the fitted u must match
the oracle's Householder lstsq and the collective (gather) transport."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, transport, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import workloads as wl
        from paper_2602_10541_b200 import dist as fdist
        from paper_2602_10541_b200 import fls
        torch.cuda.set_device(0)
        p = wl.make_problem(name, "mini")
        W, b = p.parity_features()
        F, R = p.n_features, p.n_rows
        a, e = wl.shard_range(R, rank, world)
        ctx = fls.Context(0)
        blocks = [fls.Block(torch.from_numpy(blk.X).cuda(), blk.terms, blk.weight,
                            torch.from_numpy(blk.values).cuda(),
                            torch.from_numpy(blk.fields).cuda() if blk.fields is not None else None)
                  for blk in p.blocks]
        Wd, bd = torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda()
        Ab, lda = fls.fls_assemble(ctx, Wd, bd, blocks, row_begin=a, row_end=e)
        beta, res = fdist.tsqr_solve(Ab, e - a, lda, F, ridge_rel=p.ridge_rel, ctx=ctx,
                                     transport=transport)
        Xt = torch.from_numpy(p.test_points(2000)).cuda()
        u = fls.fls_eval(ctx, Wd, bd, beta, Xt).cpu().numpy()
        q.put((rank, u, res, fdist.LAST_TRANSPORT))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _run(name, transport):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, transport, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(2):
        r, u, res, used = q.get(timeout=300)
        assert used == transport, (used, transport)     # no silent fallback
        out[r] = (u, res)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("name", ["c1_poisson1d", "c5_biharm3d"])
def test_tsqr_p2p_matches_oracle_and_collective(name):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle
    import workloads as wl
    p2p = _run(name, "p2p")
    col = _run(name, "collective")
    p = wl.make_problem(name, "mini")
    W, b = p.parity_features()
    Ao, ro, _ = oracle.assemble(W, b, p.blocks, want_scale=False)
    beta_o, _, _ = oracle.lstsq(Ao, ro, ridge_rel=p.ridge_rel)
    u_o = oracle.evaluate(W, b, beta_o, p.test_points(2000))
    for r in (0, 1):
        u = p2p[r][0]
        assert np.linalg.norm(u - u_o) / np.linalg.norm(u_o) <= 1e-6
        assert np.linalg.norm(u - col[r][0]) / np.linalg.norm(u_o) <= 1e-9
    assert abs(p2p[0][1] - col[0][1]) <= 1e-9 * max(abs(col[0][1]), 1e-300)


def test_ipc_errors():
    """an invalid IPC handle maps to FLS_ECUDA; NULL arguments to FLS_EINVAL"""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2602_10541_b200 import fls
    ctx = fls.Context(0)
    with pytest.raises(fls.FlsError, match="ECUDA"):
        fls.fls_ipc_open(ctx, bytes(64))
    t = torch.zeros(1000, dtype=torch.float64, device="cuda")
    h, off = fls.fls_ipc_handle(ctx, t[10:])
    assert len(h) == 64 and off >= 80 and off % 8 == 0      # offset of t[10:] in its allocation
