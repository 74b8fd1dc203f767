"""The multi-rank solve inside libfls (csrc/fls_comm.cu).

One GPU is available, so:
  - the NCCL control plane runs as a world-size-1 communicator (fls_comm_init) with the TSQR
    path forced -- local QR, the factor exchange (peer-memory stores into the root's stack, or
    grouped ncclSend/ncclRecv to itself), the root's stacked solve, the beta broadcast -- and
    through torch.distributed's NCCL process group (dist.attach_comm);
  - the peer-memory transport across PROCESSES runs with 2 and 3 processes sharing GPU 0 and
    the host-callback control plane over gloo (NCCL refuses two ranks on one device): rank r's
    R-extraction kernel stores into rank 0's CUDA-IPC-mapped buffer.  No kernel waits on another
    process's kernel -- every cross-rank wait is a host allgather;
  - the fallbacks: FLS_TEST_NO_IPC=1 makes the root's IPC export fail -> AUTO falls back to
    NCCL; with a host control plane (no NCCL) every rank gets FLS_EUNSUPPORTED, none hangs.
Every solve is checked against the single-process dense fls_solve of the same matrix and the
oracle's Householder lstsq (fitted u, reading A17)."""
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


def _blocks(p):
    from paper_2602_10541_b200 import fls
    return [fls.Block(torch.from_numpy(blk.X).cuda(), blk.terms, blk.weight,
                      torch.from_numpy(blk.values).cuda(),
                      torch.from_numpy(blk.fields).cuda() if blk.fields is not None else None)
            for blk in p.blocks]


def _oracle_u(p, n_test=2000):
    import oracle
    W, b = p.parity_features()
    Ao, ro, _ = oracle.assemble(W, b, p.blocks, want_scale=False)
    beta_o, _, _ = oracle.lstsq(Ao, ro, ridge_rel=p.ridge_rel)
    return oracle.evaluate(W, b, beta_o, p.test_points(n_test))


def _dense(ctx, p, Wd, bd, blocks):
    """single-process reference: one QR of the whole [A | b] (ridge rows appended locally)"""
    from paper_2602_10541_b200 import fls
    F, R = p.n_features, p.n_rows
    Ab, lda = fls.fls_assemble(ctx, Wd, bd, blocks, extra_rows=F if p.ridge_rel > 0 else 0)
    return fls.fls_solve(ctx, Ab, R, lda, F, p.ridge_rel)


@pytest.mark.parametrize("transport", ["p2p", "nccl", "auto"])
@pytest.mark.parametrize("name", ["c1_poisson1d", "c5_biharm3d"])
def test_nccl_comm_world1_forced_tsqr(name, transport):
    import workloads as wl
    from paper_2602_10541_b200 import fls
    p = wl.make_problem(name, "mini")
    W, b = p.parity_features()
    F, R = p.n_features, p.n_rows
    ctx = fls.Context(0)
    Wd, bd = torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda()
    blocks = _blocks(p)
    beta_d, res_d = _dense(ctx, p, Wd, bd, blocks)
    fls.fls_comm_init(ctx, fls.fls_comm_unique_id(), 1, 0)
    assert fls.fls_comm_info(ctx)[:2] == (1, 0)
    fls.fls_comm_config(ctx, transport, force_tsqr=True)
    Ab, lda = fls.fls_assemble(ctx, Wd, bd, blocks)           # no ridge rows needed: the root adds them
    beta, res = fls.fls_solve(ctx, Ab, R, lda, F, p.ridge_rel)
    assert fls.fls_comm_info(ctx)[2] == ("nccl" if transport == "nccl" else "p2p")
    Xt = torch.from_numpy(p.test_points(2000)).cuda()
    u = fls.fls_eval(ctx, Wd, bd, beta, Xt).cpu().numpy()
    u_d = fls.fls_eval(ctx, Wd, bd, beta_d, Xt).cpu().numpy()
    u_o = _oracle_u(p)
    assert np.linalg.norm(u - u_o) / np.linalg.norm(u_o) <= 1e-6
    assert np.linalg.norm(u - u_d) / np.linalg.norm(u_d) <= 1e-9
    assert abs(res - res_d) <= 1e-9 * max(abs(res_d), 1e-2)
    ctx.close()


def test_nccl_comm_world1_ipc_export_failure_falls_back_to_nccl(monkeypatch):
    import workloads as wl
    from paper_2602_10541_b200 import fls
    monkeypatch.setenv("FLS_TEST_NO_IPC", "1")
    p = wl.make_problem("c1_poisson1d", "mini")
    W, b = p.parity_features()
    F, R = p.n_features, p.n_rows
    ctx = fls.Context(0)
    Wd, bd = torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda()
    fls.fls_comm_init(ctx, fls.fls_comm_unique_id(), 1, 0)
    fls.fls_comm_config(ctx, "auto", force_tsqr=True)
    Ab, lda = fls.fls_assemble(ctx, Wd, bd, _blocks(p))
    beta, _ = fls.fls_solve(ctx, Ab, R, lda, F, 0.0)
    assert fls.fls_comm_info(ctx)[2] == "nccl"
    fls.fls_comm_config(ctx, "p2p", force_tsqr=True)          # P2P only: a clean error, no hang
    Ab, lda = fls.fls_assemble(ctx, Wd, bd, _blocks(p))
    with pytest.raises(fls.FlsError, match="EUNSUPPORTED"):
        fls.fls_solve(ctx, Ab, R, lda, F, 0.0)
    u = fls.fls_eval(ctx, Wd, bd, beta, torch.from_numpy(p.test_points(2000)).cuda()).cpu().numpy()
    u_o = _oracle_u(p)
    assert np.linalg.norm(u - u_o) / np.linalg.norm(u_o) <= 1e-6
    ctx.close()


def test_comm_argument_errors():
    from paper_2602_10541_b200 import fls
    ctx = fls.Context(0)
    with pytest.raises(fls.FlsError, match="EINVAL"):
        fls.fls_comm_config(ctx, "auto")                       # no communicator yet
    fls.fls_comm_init_host(ctx, 1, 0, lambda data: data)
    with pytest.raises(fls.FlsError, match="EINVAL"):
        fls.fls_comm_init_host(ctx, 1, 0, lambda data: data)   # already attached
    with pytest.raises(fls.FlsError, match="EINVAL"):
        fls.fls_comm_config(ctx, "nccl")                       # host control plane has no NCCL
    fls.fls_comm_destroy(ctx)
    with pytest.raises(fls.FlsError, match="EINVAL"):
        fls.fls_comm_init(ctx, bytes(128), 2, 2)               # rank out of range
    # a failing host callback surfaces as FLS_ENCCL, not a hang or a crash
    fls.fls_comm_init_host(ctx, 1, 0, lambda data: b"")
    fls.fls_comm_config(ctx, "p2p", force_tsqr=True)
    M = torch.randn(40 * 9, dtype=torch.float64, device="cuda")
    with pytest.raises(fls.FlsError, match="ENCCL"):
        fls.fls_solve(ctx, M, 40, 40, 8, 0.0)
    ctx.close()


def test_torch_nccl_group_world1_through_dist():
    """dist.attach_comm on a real NCCL process group: libfls's unique id broadcast through the
    group, fls_comm_init, forced TSQR -- the NCCL branches bench.py uses at N > 1"""
    import torch.distributed as dist
    import workloads as wl
    from paper_2602_10541_b200 import dist as fdist
    from paper_2602_10541_b200 import fls
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_port()}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    try:
        p = wl.make_problem("c5_biharm3d", "mini")
        W, b = p.parity_features()
        F, R = p.n_features, p.n_rows
        ctx = fls.Context(0)
        Wd, bd = torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda()
        assert fdist.attach_comm(ctx, None, force_tsqr=True) == "nccl"
        Ab, lda = fls.fls_assemble(ctx, Wd, bd, _blocks(p))
        beta, res = fdist.tsqr_solve(Ab, R, lda, F, ridge_rel=p.ridge_rel, ctx=ctx)
        assert fdist.LAST_TRANSPORT == "p2p"
        u = fls.fls_eval(ctx, Wd, bd, beta, torch.from_numpy(p.test_points(2000)).cuda()).cpu().numpy()
        u_o = _oracle_u(p)
        assert np.linalg.norm(u - u_o) / np.linalg.norm(u_o) <= 1e-6
        # the host allgather over the NCCL group (device tensors) returns rank-order bytes
        assert fdist.host_allgather()(b"abc") == b"abc"
        ctx.close()
    finally:
        dist.destroy_process_group()


def _worker(rank, world, port, name, env, q, shards=None):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), **env)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import workloads as wl
        from paper_2602_10541_b200 import dist as fdist
        from paper_2602_10541_b200 import fls
        torch.cuda.set_device(0)
        p = wl.make_problem(name, "mini")
        W, b = p.parity_features()
        F, R = p.n_features, p.n_rows
        a, e = shards[rank] if shards else wl.shard_range(R, rank, world)
        ctx = fls.Context(0)
        Wd, bd = torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda()
        blocks = _blocks(p)
        if os.environ.get("NAN_ON_RANK") == str(rank):   # a pending FLS_ENONFINITE on this rank
            blocks[0].X[3, 0] = float("nan")
        if e > a:
            Ab, lda = fls.fls_assemble(ctx, Wd, bd, blocks, row_begin=a, row_end=e)
        else:                       # a rank without rows still takes part in the solve
            lda = 4
            Ab = torch.zeros(((F + 1) * lda,), dtype=torch.float64, device="cuda")
        try:
            beta, res = fdist.tsqr_solve(Ab, e - a, lda, F, ridge_rel=p.ridge_rel, ctx=ctx)
        except fls.FlsError as err:
            q.put((rank, None, err.name, None))
            return
        Xt = torch.from_numpy(p.test_points(2000)).cuda()
        u = fls.fls_eval(ctx, Wd, bd, beta, Xt).cpu().numpy()
        q.put((rank, u, res, fdist.LAST_TRANSPORT))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _run(name, world, env=None, shards=None):
    import torch.multiprocessing as mp
    mctx = mp.get_context("spawn")
    q = mctx.Queue()
    port = _port()
    procs = [mctx.Process(target=_worker, args=(r, world, port, name, env or {}, q, shards))
             for r in range(world)]
    for pr in procs:
        pr.start()
    out = {}
    for _ in range(world):
        r, u, res, used = q.get(timeout=300)
        out[r] = (u, res, used)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    return out


@pytest.mark.parametrize("name,world", [("c1_poisson1d", 2), ("c5_biharm3d", 2), ("c1_poisson1d", 3)])
def test_p2p_tsqr_across_processes_matches_dense_and_oracle(name, world):
    import workloads as wl
    from paper_2602_10541_b200 import fls
    out = _run(name, world)
    p = wl.make_problem(name, "mini")
    W, b = p.parity_features()
    ctx = fls.Context(0)
    Wd, bd = torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda()
    beta_d, res_d = _dense(ctx, p, Wd, bd, _blocks(p))
    u_d = fls.fls_eval(ctx, Wd, bd, beta_d, torch.from_numpy(p.test_points(2000)).cuda()).cpu().numpy()
    u_o = _oracle_u(p)
    for r in range(world):
        u, res, used = out[r]
        assert used == "p2p"
        assert np.linalg.norm(u - u_o) / np.linalg.norm(u_o) <= 1e-6
        assert np.linalg.norm(u - u_d) / np.linalg.norm(u_d) <= 1e-9
        assert np.array_equal(u, out[0][0]) and res == out[0][1]   # replicated
    # the residual norm is a rounding-level number on C1 (~1e-12): compare on the rhs's scale
    assert abs(out[0][1] - res_d) <= 1e-9 * max(abs(res_d), 1e-2)
    ctx.close()


def test_p2p_tsqr_uneven_shards_trapezoidal_and_empty_rank():
    """rank 0 holds 200 rows (< F + 1 = 501: an upper-TRAPEZOIDAL factor), rank 1 the rest, rank 2
    none at all -- the stack is padded to kmax rows, the empty rank sends zeros, every rank gets
    the same beta, equal to the dense solve's"""
    import workloads as wl
    from paper_2602_10541_b200 import fls
    p = wl.make_problem("c1_poisson1d", "mini")
    R = p.n_rows
    out = _run("c1_poisson1d", 3, shards=[(0, 200), (200, R), (R, R)])
    W, b = p.parity_features()
    ctx = fls.Context(0)
    Wd, bd = torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda()
    beta_d, _ = _dense(ctx, p, Wd, bd, _blocks(p))
    u_d = fls.fls_eval(ctx, Wd, bd, beta_d, torch.from_numpy(p.test_points(2000)).cuda()).cpu().numpy()
    u_o = _oracle_u(p)
    for r in range(3):
        u, res, used = out[r]
        assert used == "p2p"
        assert np.linalg.norm(u - u_o) / np.linalg.norm(u_o) <= 1e-6
        assert np.linalg.norm(u - u_d) / np.linalg.norm(u_d) <= 1e-9
        assert np.array_equal(u, out[0][0])
    ctx.close()


def test_pending_error_on_one_rank_is_returned_on_every_rank():
    """rank 1's assembly saw a NaN (FLS_ENONFINITE pending at its fls_solve): the status is agreed
    with the peers inside the solve -- every rank returns an error, none waits forever"""
    out = _run("c1_poisson1d", 2, {"NAN_ON_RANK": "1"}, shards=[(0, 2), (2, 1002)])
    assert out[1][1] == "FLS_ENONFINITE" and out[0][1] == "FLS_ENONFINITE"


@pytest.mark.parametrize("mode", ["1", "2"])
def test_p2p_unavailable_without_nccl_errors_on_every_rank(mode):
    """the root cannot export its stack (mode 1, e.g. a VMM allocator) or a peer cannot map it
    (mode 2, e.g. no peer access): with a host control plane there is no NCCL to fall back to,
    so every rank returns FLS_EUNSUPPORTED -- none is left waiting"""
    out = _run("c1_poisson1d", 2, {"FLS_TEST_NO_IPC": mode})
    assert out[0][1] == out[1][1] == "FLS_EUNSUPPORTED"


def test_ipc_errors():
    """an invalid IPC handle maps to FLS_ECUDA; NULL arguments to FLS_EINVAL; opening a handle
    this process exported itself is refused by CUDA (FLS_ECUDA)"""
    from paper_2602_10541_b200 import fls
    ctx = fls.Context(0)
    with pytest.raises(fls.FlsError, match="ECUDA"):
        fls.fls_ipc_open(ctx, bytes(64))
    t = torch.zeros(1000, dtype=torch.float64, device="cuda")
    h, off = fls.fls_ipc_handle(ctx, t[10:])
    assert len(h) == 64 and off >= 80 and off % 8 == 0      # offset of t[10:] in its allocation
    with pytest.raises(fls.FlsError, match="ECUDA"):
        fls.fls_ipc_open(ctx, h)


def test_failed_runtime_call_does_not_poison_the_next_launch():
    """a CUDA failure inside libfls (here: opening this process's own IPC handle) resets the
    runtime's last-error state, so the next kernel launch succeeds"""
    from paper_2602_10541_b200 import fls
    ctx = fls.Context(0)
    t = torch.zeros(64, dtype=torch.float64, device="cuda")
    h, _ = fls.fls_ipc_handle(ctx, t)
    with pytest.raises(fls.FlsError, match="ECUDA"):
        fls.fls_ipc_open(ctx, h)
    W, b = fls.fls_features(ctx, 2, 16, 1.0, 0)     # launches a kernel, checks cudaGetLastError
    fls.fls_sync(ctx)
    ctx.close()
