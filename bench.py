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

Launch contract: one rank per GPU.  Under a launcher (WORLD_SIZE set) the
world size must equal --gpus; without one, --gpus N > 1 re-launches this script under
torch.distributed.run with N ranks (and exits 2 if the node has fewer than N GPUs).  n_gpus in
the JSON line is the number of distinct devices behind the ranks (checked == ranks).

Timing: W warm-up steps, then K steps bracketed by barrier + cuda.synchronize, CUDA events on
the ctx stream, max over ranks.  The output (137 GB) is >1000x L2, so every step streams past
L2 (no flush needed).  The dominant kernel's duration comes from libfls's own event pairs
around each assembly launch (fls_ctx_timing).  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import datetime
import json
import math
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
        if dist.is_initialized():
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    t = torch.tensor([sum(times) / len(times)], dtype=torch.float64, device=_cdev())
    if dist.is_initialized():
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


def e2e_device_measure(args, eng):
    """The metric end to end with A kept where the solve consumes it (device memory): every step
    copies this rank's inputs (points, coefficient fields, rhs values) from pinned host memory,
    runs the bench's call (fls_features_assemble) into the device [A | b], and reads the step's
    rhs column back to pinned host memory (the device-resident workflow: assemble, then solve
    on the GPU).  Reported beside `e2e` (every entry to the host), not instead of it."""
    import torch
    import torch.distributed as dist
    from paper_2602_10541_b200 import fls

    p, a, e = eng.p, eng.a, eng.e
    F, d, n_local, lda = p.n_features, p.dim, eng.n_local, eng.lda
    pairs, blocks, h2d = [], [], 0
    for blk, o in zip(p.blocks, p.block_offsets()):
        lo, hi = max(a, o), min(e, o + blk.n)
        if hi <= lo:
            continue
        sl = slice(lo - o, hi - o)
        hx = torch.from_numpy(np.ascontiguousarray(blk.X[sl])).pin_memory()
        hv = torch.from_numpy(np.ascontiguousarray(blk.values[sl])).pin_memory()
        hf = (torch.from_numpy(np.ascontiguousarray(blk.fields[sl])).pin_memory()
              if blk.fields is not None else None)
        dx, dv = torch.empty_like(hx, device="cuda"), torch.empty_like(hv, device="cuda")
        df = torch.empty_like(hf, device="cuda") if hf is not None else None
        pairs += [(dx, hx), (dv, hv)] + ([(df, hf)] if hf is not None else [])
        h2d += 8 * (hx.numel() + hv.numel() + (hf.numel() if hf is not None else 0))
        blocks.append(fls.Block(dx, blk.terms, blk.weight, dv, df))
    bset = fls.BlockSet(blocks, d)
    rhs_h = torch.empty((n_local,), dtype=torch.float64).pin_memory()
    rhs_d = eng.Ab[F * lda: F * lda + n_local]

    def step():
        for dv_, hv_ in pairs:
            dv_.copy_(hv_, non_blocking=True)
        fls.fls_features_assemble(eng.ctx, d, F, p.sigma, p.seed, bset, W=eng.W, b=eng.b, A=eng.Ab,
                                  lda=lda)
        rhs_h.copy_(rhs_d, non_blocking=True)

    step()
    torch.cuda.synchronize()
    times = []
    for _ in range(max(2, args.e2e_steps)):
        if dist.is_initialized():
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step()
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    t = torch.tensor([sum(times) / len(times)], dtype=torch.float64, device=_cdev())
    if dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    s_step = float(t.item())
    return {"value": p.n_rows * F / s_step, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": 8 * n_local, "s_per_step": s_step, "steps": len(times),
            "api": "fls_features_assemble (device [A | b]; inputs H2D, rhs D2H every step)"}


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
        if torch.distributed.is_initialized():
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
    if torch.distributed.is_initialized():
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


# ------------------------------------------------------------------------------------------------
# per-config block: BASELINE.json configs 1-4 on the same GPU (rank 0, N = 1)
# ------------------------------------------------------------------------------------------------
def per_config(names=("c1_poisson1d", "c2_poisson2d", "c3_poisson5d", "c4_heat2d", "c5_biharm3d"),
               budget_s=60.0, known_solves=None):
    """For each config: the bench's step (fls_features_assemble) captured in a CUDA graph of 10
    consecutive steps and replayed (the launch-latency-bound C1/C2 measured without host
    gaps) -> steady-state entries/s and fraction of the copy peak, over the short window and
    again over >= 0.5 s (`sustained`: what the board's power limiter allows); the single-shot latency
    (host call -> kernels done); the end-to-end solve by phase (known_solves: results already
    measured in this run, e.g. the headline workload's, reused instead of re-solved).  Bounded to
    about budget_s."""
    import torch
    import workloads as wl
    from paper_2602_10541_b200 import fls

    hbm_peak, _ = _peaks()
    out = {}
    t_start = time.perf_counter()
    for name in names:
        if time.perf_counter() - t_start > budget_s:
            out[name] = {"skipped": f"time budget of {budget_s:.0f} s spent"}
            continue
        p = wl.make_problem(name, "full")
        F, R, d = p.n_features, p.n_rows, p.dim
        ctx = fls.Context()
        s = torch.cuda.Stream()
        ctx.set_stream(s)
        bset = fls.BlockSet([fls.Block(torch.from_numpy(blk.X).cuda(), blk.terms, blk.weight,
                                       torch.from_numpy(blk.values).cuda(),
                                       torch.from_numpy(blk.fields).cuda()
                                       if blk.fields is not None else None)
                             for blk in p.blocks], d)
        lda = fls.round_up(R, 4)
        Ab = torch.empty(((F + 1) * lda,), dtype=torch.float64, device="cuda")
        W = torch.empty((F, d), dtype=torch.float64, device="cuda")
        b = torch.empty((F,), dtype=torch.float64, device="cuda")

        def step():
            fls.fls_features_assemble(ctx, d, F, p.sigma, p.seed, bset, W=W, b=b, A=Ab, lda=lda)

        reps = max(5, min(2000, int(2e10 / (R * F))))
        with torch.cuda.stream(s):
            for _ in range(3):
                step()
            torch.cuda.synchronize()
            singles = []
            for _ in range(5):
                t0 = time.perf_counter()
                step()
                torch.cuda.synchronize()
                singles.append(1e6 * (time.perf_counter() - t0))
            # steady state: a CUDA graph holding `per_graph` consecutive steps, replayed
            per_graph = 10 if reps >= 100 else 1
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(per_graph):
                    step()
            for _ in range(3):
                g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(s)
            for _ in range(max(1, reps // per_graph)):
                g.replay()
            e1.record(s)
            torch.cuda.synchronize()
            window_ms = e0.elapsed_time(e1)
            # the window above is short (tens of ms): the board's power limiter (sw_power_cap)
            # reacts over ~0.1-1 s, so the HBM-heavy configs are re-timed over >= 0.5 s
            n_sus = max(1, reps // per_graph)
            if window_ms < 400.0:
                n_sus = max(1, int(math.ceil(n_sus * 500.0 / max(window_ms, 1e-3))))
            e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e2.record(s)
            for _ in range(n_sus):
                g.replay()
            e3.record(s)
            torch.cuda.synchronize()
            sus_window_ms = e2.elapsed_time(e3)
        fls.fls_sync(ctx)
        ms = window_ms / (max(1, reps // per_graph) * per_graph)
        ms_sus = sus_window_ms / (n_sus * per_graph)
        del g, Ab
        ctx.close()
        torch.cuda.empty_cache()

        class A_:
            workload = name
        sol = (known_solves or {}).get(name) or solve_measure(A_, 1, 0, 0)
        out[name] = {"rows": R, "features": F, "entries": R * F, "reps": reps,
                     "steps_per_graph": per_graph,
                     "launches_per_step": "1 (fused features + records in the assembly CTAs)"
                                          if R * F <= (1 << 22) else "2 (features + prefactors, assembly)",
                     "graph_us_per_step": 1e3 * ms, "entries_per_s": R * F / (ms / 1e3),
                     "hbm_write_gbs": 8.0 * R * (F + 1) / (ms / 1e3) / 1e9,
                     "frac_of_copy_peak": 8.0 * R * F / (ms / 1e3) / 1e9 / hbm_peak,
                     "window_ms": window_ms,
                     "sustained": {"window_ms": sus_window_ms, "graph_us_per_step": 1e3 * ms_sus,
                                   "frac_of_copy_peak": 8.0 * R * F / (ms_sus / 1e3) / 1e9 / hbm_peak},
                     "single_shot_us": statistics.median(singles),
                     "solve_ms": {k: sol[k] for k in ("ms", "features_ms", "assemble_ms",
                                                      "lstsq_ms", "eval_ms")},
                     "qr_tflops": sol["qr_tflops"],
                     "rel_l2_vs_u_star": sol.get("rel_l2_vs_u_star")}
    return out


# ------------------------------------------------------------------------------------------------
# the engine: everything that touches the GPU (bench orchestration below is engine-agnostic so
# the multi-rank contract -- spawn, one device per rank, barrier + max-over-ranks timing, one
# JSON line -- is testable on CPU with an injected engine, tests/test_bench_cpu.py)
# ------------------------------------------------------------------------------------------------
class FlsEngine:
    backend = "nccl"

    @staticmethod
    def device_count() -> int:
        import torch
        return torch.cuda.device_count()

    def __init__(self, args, world, rank, local):
        import torch
        import workloads as wl
        from paper_2602_10541_b200 import fls
        self.torch, self.fls, self.args = torch, fls, args
        self.world, self.rank, self.local = world, rank, local
        torch.cuda.set_device(local)
        kw = {"n_int": args.rows} if args.rows else {}
        if args.scaling == "weak":
            base_rows = args.rows or wl.FULL[args.workload]["n_int"]
            kw["n_int"] = base_rows * world
        p = wl.make_problem(args.workload, "full", **kw)
        self.p = p
        F, R, d = p.n_features, p.n_rows, p.dim
        a, e = wl.shard_range(R, rank, world)
        self.a, self.e, self.n_local = a, e, e - a
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
        self.ctx = fls.Context(local)
        self.bset = fls.BlockSet(blocks, d)
        self.row_major = args.layout == "row"
        n_local = self.n_local
        self.lda = fls.round_up(F, 2) if self.row_major else fls.round_up(n_local, 4)
        self.Ab = torch.empty(((n_local if self.row_major else F + 1) * self.lda,),
                              dtype=torch.float64, device="cuda")
        self.rhs = torch.empty((n_local,), dtype=torch.float64, device="cuda") if self.row_major else None
        self.W = torch.empty((F, d), dtype=torch.float64, device="cuda")
        self.b = torch.empty((F,), dtype=torch.float64, device="cuda")
        # per step: one fused features + prefactor launch (plus one prefactor launch per <= 4
        # blocks when more than 4 blocks); assembly launches are counted by libfls's events
        self.fixed_launches = 1 if len(blocks) <= 4 else 1 + (len(blocks) + 3) // 4
        self.entries_total = R * F
        self.clk = None

    def device_id(self) -> str:
        return str(self.torch.cuda.get_device_properties(self.local).uuid)

    def coll_device(self):
        return "cuda"

    def step(self):
        fls, p = self.fls, self.p
        self.torch.cuda.nvtx.range_push("fls step")
        if self.row_major:
            fls.fls_features_assemble(self.ctx, p.dim, p.n_features, p.sigma, p.seed, self.bset,
                                      W=self.W, b=self.b, A=self.Ab, lda=self.lda,
                                      layout=fls.FLS_ROW_MAJOR, rhs=self.rhs)
        else:
            fls.fls_features_assemble(self.ctx, p.dim, p.n_features, p.sigma, p.seed, self.bset,
                                      W=self.W, b=self.b, A=self.Ab, lda=self.lda)
        self.torch.cuda.nvtx.range_pop()

    def sync(self):
        self.fls.fls_sync(self.ctx)
        self.torch.cuda.synchronize()

    def begin_timed(self):
        self.fls.fls_sync(self.ctx)
        self.clk = ClockSampler(self.local)
        self.clk.start()
        time.sleep(0.3)                      # let nvidia-smi start sampling
        self.fls.fls_ctx_timing(self.ctx, True)
        self.ev = [self.torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def start(self):
        self.torch.cuda.synchronize()
        self.clk.mark_begin()
        self.ev[0].record(self.ctx.stream)

    def stop(self) -> float:
        self.ev[1].record(self.ctx.stream)
        self.torch.cuda.synchronize()
        self.clk.mark_end()
        return self.ev[0].elapsed_time(self.ev[1])

    def end_timed(self):
        self.clocks = self.clk.stop()
        self.fls.fls_sync(self.ctx)
        self.k_ms, self.k_launches = self.fls.fls_ctx_timing_read(self.ctx)
        self.fls.fls_ctx_timing(self.ctx, False)

    def kernel_report(self, steps):
        """this rank's dominant-kernel numbers (algorithmic bytes = 8 B per entry)"""
        p, n_local = self.p, self.n_local
        F = p.n_features
        k_ms_step = self.k_ms / steps
        achieved = 8.0 * n_local * F / (k_ms_step / 1e3) / 1e9
        return {"achieved": achieved, "bytes_per_step": 8.0 * n_local * F,
                "kernel_ms_per_step": k_ms_step,
                "kernel_ms_avg": self.k_ms / max(self.k_launches, 1),
                "launches": self.k_launches, "entries_per_s": n_local * F / (k_ms_step / 1e3)}

    def report(self, steps, ms_step, per_rank, n_gpus):
        torch, p, args = self.torch, self.p, self.args
        F, R, d = p.n_features, p.n_rows, p.dim
        hbm_peak, peak_kind = _peaks()
        mine = per_rank[self.rank]
        achieved = mine["achieved"]
        traffic = None
        tf = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tf) and args.rows is None and self.world == 1:
            try:
                traffic = json.load(open(tf)).get(args.workload, {}).get("traffic_bytes_per_launch")
            except Exception:
                traffic = None
        # FP64 co-bound (north_star: "the slower of HBM bandwidth and fp64 issue rate")
        ops = fp64_ops_per_entry(p)
        fp64 = None
        clocks = self.clocks
        if ops is not None:
            sms = torch.cuda.get_device_properties(self.local).multi_processor_count
            ach = ops * mine["entries_per_s"] / 1e12
            fp64 = {"ops_per_entry": ops, "achieved_tops": ach}
            for tag, mhz in (("max_clock", clocks.get("sm_max_mhz")), ("median_clock", clocks.get("sm_mhz"))):
                if mhz:
                    pk = sms * 64 * mhz * 1e6 / 1e12
                    fp64[f"peak_tops_{tag}"] = pk
                    fp64[f"frac_{tag}"] = ach / pk
        power = None
        pm = os.path.join(ROOT, "profiles", "r02_power_model.json")
        if not os.path.exists(pm):
            pm = os.path.join(ROOT, "profiles", "r01_power_model.json")
        if os.path.exists(pm) and p.name == "c5_biharm3d":
            try:
                m = json.load(open(pm))["model"]
                bound = m["power_bound_entries_per_s"]
                window_s = ms_step * steps / 1e3
                sustained = window_s >= 4.0
                power = {"bound": "board power (sustained windows >= 4 s)",
                         "limit_w": m["power_limit_w"], "idle_w": m["idle_w"],
                         "nj_per_entry": m["store_nj_per_entry"] + m["alu_nj_per_entry"],
                         "bound_entries_per_s_per_gpu": bound,
                         "achieved_entries_per_s_per_gpu": mine["entries_per_s"],
                         "timed_window_s": window_s,
                         # the limiter acts on a time-averaged power: over a window shorter
                         # than ~4 s the board borrows headroom, so no fraction is claimed
                         "frac": mine["entries_per_s"] / bound if sustained else None,
                         "frac_short_window": None if sustained else mine["entries_per_s"] / bound,
                         "sustained_reference": {
                             "frac": m.get("c5_assembly_frac_of_power_bound"),
                             "what": "the same kernel back to back for 4 s at 995 W of 1000 W"},
                         "source": os.path.relpath(pm, ROOT) + " (tools/power_model.py)"}
            except Exception:
                power = None
        # north_star's roofline: "the slower of HBM bandwidth and the fp64 sincos issue rate".
        # The FP64 side is the measured register-only rate of the C5 per-entry arithmetic
        # (microbench entry kernel, no memory traffic) at full clock, scaled to the SM clock
        # the timed region actually ran at (the board lowers it under sw_power_cap)
        co_bound = None
        if os.path.exists(pm) and p.name == "c5_biharm3d" and clocks.get("sm_mhz"):
            try:
                mm = json.load(open(pm))
                alu_full, mhz_full = mm["c5_alu"]["entries_per_s"], mm["c5_alu"]["clocks"]["sm_mhz"]
                alu_now = alu_full * clocks["sm_mhz"] / mhz_full
                n_ent = mine["bytes_per_step"] / 8.0
                t_hbm = mine["bytes_per_step"] / (hbm_peak * 1e9) * 1e3
                t_fp64 = n_ent / alu_now * 1e3
                t_kern = mine["kernel_ms_per_step"]
                co_bound = {"bound": "fp64" if t_fp64 > t_hbm else "hbm",
                            "t_hbm_ms": t_hbm, "t_fp64_ms_at_median_clock": t_fp64,
                            "kernel_ms": t_kern, "frac": max(t_hbm, t_fp64) / t_kern,
                            "fp64_entries_per_s_full_clock": alu_full,
                            "median_sm_mhz": clocks["sm_mhz"],
                            "source": os.path.relpath(pm, ROOT) + " (c5_alu)"}
            except Exception:
                co_bound = None
        tot_bytes = sum(r["bytes_per_step"] for r in per_rank)
        slowest = max(r["kernel_ms_per_step"] for r in per_rank)
        agg = tot_bytes / (slowest / 1e3) / 1e9
        return {
            "dtype": "f64",
            "config": {"workload": p.name, "rows": R, "features": F, "dim": d,
                       "operator": "biharmonic + 16(1+x1) u" if p.name == "c5_biharm3d" else p.name,
                       "A_bytes": 8 * R * (F + 1), "parallelism": f"rows{self.world}",
                       "rows_per_rank": [int(r["bytes_per_step"] / 8 / F) for r in per_rank],
                       "l2": f"no flush: each step writes {8e-9 * self.n_local * (F + 1):.1f} GB per "
                             f"GPU (>> the 126 MB L2)"},
            "hbm_write_gbs_all_gpus": 8.0 * R * (F + 1) / (ms_step / 1e3) / 1e9,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic,
                         "peak_kind": f"{peak_kind} copy bandwidth (MEASURED_PEAKS.json hbm_gbs)",
                         "kernel": "assemble_rm_kernel" if self.row_major else "assemble_cm_kernel",
                         "kernel_ms_avg": mine["kernel_ms_avg"], "fp64_pipe": fp64, "power": power,
                         "co_bound": co_bound,
                         "scope": "rank 0's GPU (per-GPU kernel roofline)",
                         "per_rank": [{"rank": i, "achieved": r["achieved"],
                                       "frac": r["achieved"] / hbm_peak} for i, r in enumerate(per_rank)],
                         "aggregate": {"achieved": agg, "peak": hbm_peak * n_gpus,
                                       "frac": agg / (hbm_peak * n_gpus),
                                       "note": "all ranks' algorithmic bytes / the slowest rank's "
                                               "kernel time, against n_gpus x the copy peak"}},
            "gpu_launches": self.fixed_launches * steps + mine["launches"],
            "clocks": clocks,
        }

    def extras(self, args):
        """legs after the timed region: e2e through the C ABI with host buffers, the
        end-to-end solve, per-config numbers and the CPU oracle (rank 0, N = 1)"""
        torch = self.torch
        out = {}

        def leg(key, fn):
            # at N = 1 a failing auxiliary leg is recorded and the headline line still prints;
            # at N > 1 it propagates (a rank that skipped a leg's collectives would desynchronise
            # the others)
            if self.world > 1:
                out[key] = fn()
                return
            try:
                out[key] = fn()
            except Exception as ex:  # noqa: BLE001 -- reported in the JSON line
                out[key] = {"error": f"{type(ex).__name__}: {ex}"[:300]}
                sys.stderr.write(f"bench.py: leg {key} failed: {ex}\n")

        if not args.no_e2e:
            leg("e2e_device_resident", lambda: e2e_device_measure(args, self))
        del self.Ab
        torch.cuda.empty_cache()
        if not args.no_e2e:
            leg("e2e", lambda: e2e_measure(args, self.p, self.ctx, self.W, self.b, self.a, self.e,
                                           self.world, self.local))
        if not args.no_solve and args.rows is None:
            leg("solve", lambda: solve_measure(args, self.world, self.rank, self.local))
        solve_ok = "solve" in out and "error" not in out["solve"]
        if self.world == 1 and args.rows is None and not args.no_per_config:
            leg("per_config", lambda: per_config(
                budget_s=args.per_config_budget,
                known_solves={self.p.name: out["solve"]} if solve_ok else None))
        if self.rank == 0 and self.world == 1 and not args.no_cpu:
            leg("cpu_baseline", lambda: cpu_baseline(self.p))
        return out

    def close(self):
        self.ctx.close()


def _engine_class():
    """FLS_BENCH_ENGINE=path/to/file.py:Class injects an engine (CPU tests of the multi-rank
    contract, tests/fake_bench_engine.py)"""
    spec = os.environ.get("FLS_BENCH_ENGINE")
    if not spec:
        return FlsEngine
    import importlib.util
    path, cls = spec.rsplit(":", 1)
    ms = importlib.util.spec_from_file_location("fls_bench_engine", os.path.join(ROOT, path))
    mod = importlib.util.module_from_spec(ms)
    ms.loader.exec_module(mod)
    return getattr(mod, cls)


def _free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn_ranks(args, argv) -> int:
    """`python bench.py --gpus N` without a launcher: start N ranks, one per GPU, under
    torch.distributed.run (the same launch the driver uses) and return its exit code.  Rank 0
    prints the JSON line.  Fails loudly when the node has fewer than N GPUs."""
    eng = _engine_class()
    have = eng.device_count()
    if args.gpus > have:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this node has "
                         f"{have}\n")
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__)] + list(argv)
    return subprocess.call(cmd)


def run_ranks(args) -> int:
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    eng_cls = _engine_class()
    shared = os.environ.get("FLS_BENCH_SHARED_GPU") == "1"   # test mode: ranks share GPUs
    if world != args.gpus:
        sys.stderr.write(f"bench.py: launched with WORLD_SIZE={world} but --gpus {args.gpus}\n")
        return 2
    have = eng_cls.device_count()
    if shared:
        local %= max(1, have)
    elif local >= have:
        sys.stderr.write(f"bench.py: rank {rank} has LOCAL_RANK {local} but the node has {have} GPUs\n")
        return 2
    backend = "gloo" if shared else eng_cls.backend
    # a process group whenever a launcher started us (also at world size 1: the timing
    # collectives then run through NCCL exactly as at N > 1)
    pg = "WORLD_SIZE" in os.environ and "MASTER_ADDR" in os.environ
    if pg:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    eng = eng_cls(args, world, rank, local)
    cdev = "cpu" if backend == "gloo" else eng.coll_device()
    # one device per rank: count the distinct devices behind the ranks
    ids = [eng.device_id()]
    if pg:
        ids = [None] * world
        dist.all_gather_object(ids, eng.device_id())
    n_gpus = len(set(ids))
    if n_gpus != world and not shared:
        if rank == 0:
            sys.stderr.write(f"bench.py: {world} ranks share {n_gpus} device(s); one GPU per rank "
                             f"is required\n")
        if pg:
            dist.destroy_process_group()
        return 2
    for _ in range(args.warmup):
        eng.step()
    eng.sync()
    eng.begin_timed()
    if pg:
        dist.barrier()
    eng.start()
    for _ in range(args.steps):
        eng.step()
    ms_total = eng.stop()
    if pg:
        dist.barrier()
    eng.end_timed()
    t = torch.tensor([ms_total], dtype=torch.float64, device=cdev)
    if pg:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    mine = eng.kernel_report(args.steps)
    per_rank = [mine]
    if pg:
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine)
    line = {"metric": METRIC, "value": eng.entries_total / (ms_step / 1e3), "unit": UNIT,
            "n_gpus": n_gpus, "ranks": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "data": "synthetic"}
    line.update(eng.report(args.steps, ms_step, per_rank, n_gpus))
    line.update(eng.extras(args))
    if rank == 0:
        print(json.dumps(line), flush=True)
    eng.close()
    if pg:
        dist.destroy_process_group()
    return 0


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
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
    ap.add_argument("--no-per-config", action="store_true", help="skip the C1-C4 per-config leg")
    ap.add_argument("--per-config-budget", type=float, default=60.0)
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the config's rows split over the ranks (BASELINE config 5's "
                         "sweep, default); weak: every rank keeps the config's full row count")
    ap.add_argument("--layout", default="col", choices=["col", "row"],
                    help="A layout (col = what the QR consumes; row = features contiguous)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--e2e-ring-rows", type=int, default=262144)
    ap.add_argument("--rows", type=int, default=None,
                    help="override the interior row count (profiling a reduced copy of the workload)")
    args = ap.parse_args(argv)
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if args.impl == "reference":
        return run_reference(args) or 0
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args, argv)
    return run_ranks(args)


if __name__ == "__main__":
    sys.exit(main())
