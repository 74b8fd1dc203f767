#!/usr/bin/env python
"""Benchmark of the Fast-LSQ assembly hot path (BASELINE.json metric: A-assembly entries/s and
HBM GB/s, fp64).

One STEP = one pass of the whole hot path of SURVEY §8(a) over the workload:
  a1 + a2-a8 fls_features_assemble (W, b from Philox on the device, prefactor fold,
  phase, trig, combine, weighted row blocks, rhs, streaming fp64 stores of [A | b]).
Default workload = BASELINE.json config 5 (3D biharmonic + variable-coefficient Helmholtz,
2,097,152 rows x 8,192 features = 1.718e10 entries, 137.4 GB of fp64), row-sharded over the
ranks (strong scaling: the config fixes the total rows).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fls|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Timing: W warm-up steps, then K steps bracketed by barrier + cuda.synchronize, CUDA events on
the ctx stream, max over ranks.  The output (137 GB) is >1000x L2, so every step streams past
L2 (no flush needed).  The dominant kernel's duration comes from libfls's own event pairs
around each assembly launch (fls_ctx_timing).  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import datetime
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "A-assembly entries/s (fp64)"
UNIT = "entries/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            P = json.load(f)
        return float(P["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def fp64_ops_per_entry(p):
    """FP64-pipe instructions per entry of the sin-family assembly kernel (SASS-
    checked for C5): d phase DFMA + 3 DADD rounding + f^2 + 6 DFMA polynomial + 1 DMUL (·f) +
    1 DMUL (·P) + 1 DFMA per coefficient-field group.  Row-weighted over the blocks; None when
    a block needs the sin+cos variant (mixed parity with coefficient fields)."""
    tot = 0.0
    for blk in p.blocks:
        groups = {int(f) for _, _, f in blk.terms if int(f) >= 0}
        parities = {sum(a) % 2 for a, _, _ in blk.terms}
        if groups and len(parities) > 1:
            return None
        tot += blk.n * (p.dim + 12 + len(groups))
    return tot / max(p.n_rows, 1)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region"""

    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self.proc = None
        self.t0 = self.t1 = None

    def mark_begin(self):   # host wall-clock bracket of the timed region (samples outside are
        self.t0 = datetime.datetime.now()   # idle or warm-up and are dropped when possible)

    def mark_end(self):
        self.t1 = datetime.datetime.now()

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 10:
                try:
                    ts = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f")
                except ValueError:
                    ts = None
                self.rows.append((ts, parts[1:]))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons, pw = [], 0.0, set(), []
        rows = [r for ts, r in self.rows]
        window = "sampler lifetime"
        if self.t0 and self.t1:
            inside = [r for ts, r in self.rows if ts is not None and self.t0 <= ts <= self.t1]
            if inside:
                rows, window = inside, "timed region"
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = max(mx, float(r[2]))
                pw.append(float(r[3]))
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if r[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "sm_min_mhz": min(sm) if sm else None, "power_w_max": max(pw) if pw else None,
                "power_w_median": statistics.median(pw) if pw else None,
                "reasons": sorted(reasons), "samples": len(sm), "window": window}


def cpu_baseline(problem, rows_budget_s: float = 12.0):
    """The oracle as it stands on the host cores, on a bounded row sample of the workload."""
    import oracle
    W, b = problem.parity_features()
    R = problem.n_rows
    n = 16
    best = None
    while True:
        rows = np.linspace(0, R - 1, n).astype(np.int64)
        t0 = time.perf_counter()
        oracle.assemble(W, b, problem.blocks, rows=rows, want_scale=False)
        dt = time.perf_counter() - t0
        best = (n, dt)
        if dt > rows_budget_s / 3 or n >= R:
            break
        n = min(R, n * 4)
    n, dt = best
    ent = n * problem.n_features
    cores = oracle.max_threads()
    # the same oracle on one thread (1 thread and all cores), smaller sample
    n1 = max(16, n // max(cores, 1))
    rows1 = np.linspace(0, R - 1, n1).astype(np.int64)
    oracle.set_threads(1)
    t0 = time.perf_counter()
    oracle.assemble(W, b, problem.blocks, rows=rows1, want_scale=False)
    dt1 = time.perf_counter() - t0
    oracle.set_threads(cores)
    return {"value": ent / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{n} evenly spaced rows x all {problem.n_features} features of "
                      f"{problem.name} ({ent:.3g} entries, {dt:.2f} s)",
            "value_1_thread": n1 * problem.n_features / dt1,
            "sample_1_thread": f"{n1} evenly spaced rows, {dt1:.2f} s"}


def run_reference(args):
    """--impl reference: the CPU oracle as the reference arm (tier rules), rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    import workloads as wl
    p = wl.make_problem(args.workload, "full")
    W, b = p.parity_features()
    R, F = p.n_rows, p.n_features
    n = args.ref_rows
    times = []
    for s in range(args.warmup + args.steps):
        rows = (np.arange(n, dtype=np.int64) * 7919 + s * 104729) % R
        t0 = time.perf_counter()
        oracle.assemble(W, b, p.blocks, rows=rows, want_scale=False)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
    ms = 1e3 * sum(times) / len(times)
    val = n * F / (ms / 1e3)
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": p.name, "rows": R, "features": F,
                                            "sample_rows_per_step": n},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": oracle.max_threads(),
                             "kind": "oracle",
                             "sample": f"{n} rows/step x {F} features of {p.name}"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _cdev():
    """device for the timing collectives: the GPU under NCCL, the host under gloo"""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_backend() == "gloo":
        return "cpu"
    return "cuda"


def e2e_measure(args, p, ctx, W, b, a, e, world, local):
    """The same metric through the C ABI with HOST buffers (fls_assemble_host): every step copies
    this rank's inputs (points, fields, values, W, b) from pinned host memory and every entry of
    [A | b] back to pinned host memory.  The host output is a pinned ring of `ring` rows that
    each call overwrites (a streaming consumer's view; 137 GB would not fit the host)."""
    import torch
    import torch.distributed as dist
    from paper_2602_10541_b200 import fls

    F, d = p.n_features, p.dim
    W_h = W.cpu().pin_memory()
    b_h = b.cpu().pin_memory()

    class HB:
        pass
    hblocks = []
    in_bytes_points = 0
    offs = p.block_offsets()
    for blk, o in zip(p.blocks, offs):
        h = HB()
        h.X = torch.from_numpy(blk.X).pin_memory()
        h.terms = blk.terms
        h.weight = blk.weight
        h.values = torch.from_numpy(blk.values).pin_memory()
        h.fields = torch.from_numpy(blk.fields).pin_memory() if blk.fields is not None else None
        hblocks.append(h)
        lo, hi = max(a, o), min(e, o + blk.n)
        if hi > lo:
            per = d + 1 + (blk.fields.shape[1] if blk.fields is not None else 0)
            in_bytes_points += 8 * (hi - lo) * per
    hset = fls.HostBlockSet(hblocks, d)
    n_local = e - a
    # host ring per rank shrinks with the rank count so N ranks pin at most ~17 GB in total
    ring = min(n_local, max(8192, args.e2e_ring_rows // world))
    A_h = torch.empty((F + 1) * ring, dtype=torch.float64).pin_memory()
    n_calls = (n_local + ring - 1) // ring

    def step():
        for c in range(n_calls):
            r0 = a + c * ring
            r1 = min(e, r0 + ring)
            fls.fls_assemble_host(ctx, W_h, b_h, hset, A_h, ring, A_h[F * ring:], row_begin=r0,
                                  row_end=r1)

    step()                                   # warm-up (staging allocation, first touch)
    times = []
    for _ in range(args.e2e_steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    t = torch.tensor([sum(times) / len(times)], dtype=torch.float64, device=_cdev())
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    s_step = float(t.item())
    h2d = in_bytes_points + n_calls * 8 * (F * d + F)
    d2h = 8 * n_local * (F + 1)
    # the bound of this path: plain device -> pinned-host copy bandwidth of the same link
    probe = torch.empty(min(A_h.numel(), 1 << 28), dtype=torch.float64, device="cuda")
    host = A_h[: probe.numel()]
    host.copy_(probe, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        host.copy_(probe, non_blocking=True)
    torch.cuda.synchronize()
    d2h_peak = 3 * 8 * probe.numel() / (time.perf_counter() - t0) / 1e9
    del probe
    return {"value": p.n_rows * F / s_step, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "s_per_step": s_step, "steps": args.e2e_steps,
            "api": "fls_assemble_host (C ABI, host buffers)",
            "d2h_gbs": d2h / s_step / 1e9,
            "d2h_copy_peak_gbs": d2h_peak,
            "frac_of_d2h_copy_peak": (d2h / s_step / 1e9) / d2h_peak,
            "note": f"pinned host ring of {ring} rows x {F + 1} columns, {n_calls} calls per step"}


def solve_measure(args, world, rank, local):
    """End-to-end solve (BASELINE metric "end-to-end solve ms"), per phase, Algorithm 1 lines
    1-6: features + assembly + least squares (QR; TSQR over the ranks) + eval at 10,000
    held-out points.  C5 solves its first 262,144 rows (J:configs[5]) with the tau = 1e-10
    ridge (reading A16); other workloads solve all rows."""
    import torch
    import workloads as wl
    from paper_2602_10541_b200 import dist as fdist
    from paper_2602_10541_b200 import fls

    kw = {"n_int": 262_144} if args.workload == "c5_biharm3d" else {}
    p = wl.make_problem(args.workload, "full", **kw)
    F, R, d = p.n_features, p.n_rows, p.dim
    a, e = wl.shard_range(R, rank, world)
    n_local = e - a
    offs = p.block_offsets()
    blocks = []
    for blk, o in zip(p.blocks, offs):
        lo, hi = max(a, o), min(e, o + blk.n)
        if hi <= lo:
            continue
        sl = slice(lo - o, hi - o)
        blocks.append(fls.Block(torch.from_numpy(np.ascontiguousarray(blk.X[sl])).cuda(), blk.terms,
                                blk.weight, torch.from_numpy(np.ascontiguousarray(blk.values[sl])).cuda(),
                                torch.from_numpy(np.ascontiguousarray(blk.fields[sl])).cuda()
                                if blk.fields is not None else None))
    bset = fls.BlockSet(blocks, d)
    ctx = fls.Context(local)
    Xt = torch.from_numpy(p.test_points(10_000)).cuda()
    extra = F if (p.ridge_rel > 0 and world == 1) else 0
    lda = fls.round_up(n_local + extra, 4)
    Ab = torch.empty(((F + 1) * lda,), dtype=torch.float64, device="cuda")
    st = ctx.stream
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]

    def run():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        ev[0].record(st)
        W, b = fls.fls_features(ctx, d, F, p.sigma, p.seed)
        ev[1].record(st)
        fls.fls_assemble(ctx, W, b, bset, row_begin=0, row_end=n_local, A=Ab, lda=lda)
        ev[2].record(st)
        beta, res = fdist.tsqr_solve(Ab, n_local, lda, F, ridge_rel=p.ridge_rel, ctx=ctx)
        ev[3].record(st)
        u = fls.fls_eval(ctx, W, b, beta, Xt)
        ev[4].record(st)
        torch.cuda.synchronize()
        return u, res

    run()                                   # warm-up (cuSOLVER workspace, handles)
    u, res = run()
    ph = [ev[k].elapsed_time(ev[k + 1]) for k in range(4)]
    t = torch.tensor(ph, dtype=torch.float64, device=_cdev())
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ph = [float(v) for v in t.tolist()]
    us = p.u_star(Xt.cpu().numpy())
    uh = u.cpu().numpy()
    ctx.close()
    out = {"ms": sum(ph), "features_ms": ph[0], "assemble_ms": ph[1], "lstsq_ms": ph[2],
           "eval_ms": ph[3], "rows": R, "features": F, "ridge_rel": p.ridge_rel,
           "method": "Householder QR (fls_geqrf: blocked compact-WY on cuBLAS DGEMM + cooperative leaf kernel) + trsv"
                     + (f" / TSQR over ranks ({fdist.LAST_TRANSPORT} transport)" if world > 1 else ""),
           "qr_flops": 2.0 * (R + extra) * (F + 1) ** 2 - 2.0 / 3.0 * (F + 1) ** 3,
           "resid_norm": res}
    out["qr_tflops"] = out["qr_flops"] / (ph[2] / 1e3) / 1e12
    if args.workload != "c5_biharm3d":   # C5 has no BC rows: u* is not the LS solution (A12)
        out["rel_l2_vs_u_star"] = float(np.linalg.norm(uh - us) / np.linalg.norm(us))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="fls", choices=["fls", "reference"])
    ap.add_argument("--workload", default="c5_biharm3d")
    ap.add_argument("--no-cpu", action="store_true", help="skip the oracle cpu_baseline leg")
    ap.add_argument("--ref-rows", type=int, default=1024)
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer end-to-end leg")
    ap.add_argument("--no-solve", action="store_true", help="skip the end-to-end solve leg")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's rows split over the ranks (BASELINE config 5's "
                         "sweep, default); weak: every rank keeps the config's full row count")
    ap.add_argument("--layout", default="col", choices=["col", "row"],
                    help="A layout (col = what the QR consumes; row = features contiguous)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--e2e-ring-rows", type=int, default=262144)
    ap.add_argument("--rows", type=int, default=None,
                    help="override the interior row count (profiling a reduced copy of the workload)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import workloads as wl
    from paper_2602_10541_b200 import fls

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local %= max(1, torch.cuda.device_count())      # ranks > GPUs only in the gloo test mode
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL over NVLink; FLS_DIST_BACKEND=gloo runs the multi-rank host logic with host
        # collectives (e.g. 2 ranks sharing one GPU in a test; no kernel waits on another rank)
        backend = os.environ.get("FLS_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    kw = {"n_int": args.rows} if args.rows else {}
    if args.scaling == "weak":
        # every rank keeps the config's full row count: the job is world x the config's rows
        base_rows = args.rows or wl.FULL[args.workload]["n_int"]
        kw["n_int"] = base_rows * world
    p = wl.make_problem(args.workload, "full", **kw)
    F, R, d = p.n_features, p.n_rows, p.dim
    a, e = wl.shard_range(R, rank, world)
    n_local = e - a
    # this rank's points only (inputs resident in HBM before timing)
    offs = p.block_offsets()
    blocks = []
    for blk, o in zip(p.blocks, offs):
        lo, hi = max(a, o), min(e, o + blk.n)
        if hi <= lo:
            continue
        sl = slice(lo - o, hi - o)
        blocks.append(fls.Block(torch.from_numpy(np.ascontiguousarray(blk.X[sl])).cuda(), blk.terms,
                                blk.weight, torch.from_numpy(np.ascontiguousarray(blk.values[sl])).cuda(),
                                torch.from_numpy(np.ascontiguousarray(blk.fields[sl])).cuda()
                                if blk.fields is not None else None))
    ctx = fls.Context(local)
    bset = fls.BlockSet(blocks, d)
    row_major = args.layout == "row"
    lda = fls.round_up(F, 2) if row_major else fls.round_up(n_local, 4)
    Ab = torch.empty(((n_local if row_major else F + 1) * lda,), dtype=torch.float64, device="cuda")
    rhs = torch.empty((n_local,), dtype=torch.float64, device="cuda") if row_major else None
    W = torch.empty((F, d), dtype=torch.float64, device="cuda")
    b = torch.empty((F,), dtype=torch.float64, device="cuda")
    # per step: one fused features + prefactor launch (plus one prefactor launch per <= 4 blocks
    # when more than 4 blocks); assembly launches are counted by libfls's own timing events
    # (one per batch of blocks sharing a kernel variant)
    launches_per_step_fixed = 1 if len(blocks) <= 4 else 1 + (len(blocks) + 3) // 4

    def step():
        torch.cuda.nvtx.range_push("fls step")   # NVTX: one range per step for nsys timelines
        if row_major:
            fls.fls_features_assemble(ctx, d, F, p.sigma, p.seed, bset, W=W, b=b, A=Ab, lda=lda,
                                      layout=fls.FLS_ROW_MAJOR, rhs=rhs)
        else:
            fls.fls_features_assemble(ctx, d, F, p.sigma, p.seed, bset, W=W, b=b, A=Ab, lda=lda)
        torch.cuda.nvtx.range_pop()

    for _ in range(args.warmup):
        step()
    fls.fls_sync(ctx)
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)                      # let nvidia-smi start sampling
    fls.fls_ctx_timing(ctx, True)
    st = ctx.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clk.mark_begin()
    e0.record(st)
    for _ in range(args.steps):
        step()
    e1.record(st)
    torch.cuda.synchronize()
    clk.mark_end()
    if world > 1:
        dist.barrier()
    clocks = clk.stop()
    fls.fls_sync(ctx)
    ms_total = e0.elapsed_time(e1)
    k_ms, k_launches = fls.fls_ctx_timing_read(ctx)
    fls.fls_ctx_timing(ctx, False)
    t = torch.tensor([ms_total], dtype=torch.float64, device=_cdev())
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    entries = R * F
    value = entries / (ms_step / 1e3)

    # roofline of the dominant kernel (assembly): algorithmic bytes = 8 B x entries per launch
    hbm_peak, peak_kind = _peaks()
    k_avg_ms = k_ms / max(k_launches, 1)
    # algorithmic bytes of all assembly launches of one step / their summed time per step
    k_ms_step = k_ms / args.steps
    achieved = 8.0 * n_local * F / (k_ms_step / 1e3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf) and args.rows is None and world == 1:
        try:
            traffic = json.load(open(tf)).get(args.workload, {}).get("traffic_bytes_per_launch")
        except Exception:
            traffic = None
    # the FP64 co-bound (north_star: "the slower of HBM bandwidth and fp64 issue rate"): FP64-pipe
    # lane-ops per second vs 148 SMs x 64 FP64 lanes/clk at the max and the median loaded clock
    ops = fp64_ops_per_entry(p)
    fp64 = None
    if ops is not None:
        sms = torch.cuda.get_device_properties(local).multi_processor_count
        ach = ops * n_local * F / (k_ms_step / 1e3) / 1e12
        fp64 = {"ops_per_entry": ops, "achieved_tops": ach}
        for tag, mhz in (("max_clock", clocks.get("sm_max_mhz")), ("median_clock", clocks.get("sm_mhz"))):
            if mhz:
                pk = sms * 64 * mhz * 1e6 / 1e12
                fp64[f"peak_tops_{tag}"] = pk
                fp64[f"frac_{tag}"] = ach / pk
    # the binding roofline under sustained load: board power (profiles/r01_power_model.json,
    # tools/power_model.py: idle power + measured energy per entry of the store pattern and of the
    # per-entry arithmetic, each probed alone) -> entries/s <= (P_limit - P_idle) / (E_st + E_alu)
    power = None
    pm = os.path.join(ROOT, "profiles", "r01_power_model.json")
    if os.path.exists(pm) and p.name == "c5_biharm3d":
        try:
            m = json.load(open(pm))["model"]
            bound = m["power_bound_entries_per_s"]
            power = {"bound": "board power", "limit_w": m["power_limit_w"], "idle_w": m["idle_w"],
                     "nj_per_entry": m["store_nj_per_entry"] + m["alu_nj_per_entry"],
                     "bound_entries_per_s_per_gpu": bound,
                     "achieved_entries_per_s_per_gpu": n_local * F / (k_ms_step / 1e3),
                     "frac": n_local * F / (k_ms_step / 1e3) / bound,
                     "source": "profiles/r01_power_model.json (tools/power_model.py)",
                     "note": "a 20-step run can read above 1.0: the board's limiter acts on a "
                             "time-averaged power, so short runs borrow headroom; run back to "
                             "back for 4 s the kernel sits at 0.99 (995 W of 1000 W)"}
        except Exception:
            power = None
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": p.name, "rows": R, "features": F, "dim": d,
                   "operator": "biharmonic + 16(1+x1) u" if p.name == "c5_biharm3d" else p.name,
                   "A_bytes": 8 * R * (F + 1), "parallelism": f"rows{world}",
                   "l2": f"no flush: each step writes {8e-9 * n_local * (F + 1):.1f} GB per GPU "
                         f"(>> the 126 MB L2)"},
        "hbm_write_gbs_all_gpus": 8.0 * R * (F + 1) / (ms_step / 1e3) / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic,
                     "peak_kind": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
                     "kernel": "assemble_rm_kernel" if row_major else "assemble_cm_kernel",
                     "kernel_ms_avg": k_avg_ms, "fp64_pipe": fp64, "power": power,
                     "scope": "rank 0's GPU (per-GPU kernel roofline)"},
        "gpu_launches": launches_per_step_fixed * args.steps + k_launches,
        "clocks": clocks,
    }
    # ---------------------------------------------------------------- end to end (host buffers)
    del Ab
    torch.cuda.empty_cache()
    if not args.no_e2e:
        line["e2e"] = e2e_measure(args, p, ctx, W, b, a, e, world, local)
    if not args.no_solve and args.rows is None:
        line["solve"] = solve_measure(args, world, rank, local)
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline(p)
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
