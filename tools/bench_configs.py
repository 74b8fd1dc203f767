"""Per-config table for BASELINE.md §4: all five BASELINE.json configs on one GPU.

For each config: steady-state assembly throughput (features + assembly captured once in a CUDA
graph and replayed, so the latency-bound C1/C2 are measured without host launch gaps, plus the
single-shot latency), the end-to-end solve by phase, fitted-u parity against the oracle
(in-run for C1/C2, tests/golden/oracle_u_<cfg>.npz artifacts for C3-C5 when present), and the
oracle's own assembly rate on sampled rows (1 thread and all host threads).

    python tools/bench_configs.py [cfg ...] > profiles/r01_configs.jsonl
"""
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workloads as wl  # noqa: E402
from bench import ClockSampler, _peaks  # noqa: E402
from paper_2602_10541_b200 import fls  # noqa: E402


def dev_blocks(p):
    return [fls.Block(torch.from_numpy(blk.X).cuda(), blk.terms, blk.weight,
                      torch.from_numpy(blk.values).cuda(),
                      torch.from_numpy(blk.fields).cuda() if blk.fields is not None else None)
            for blk in p.blocks]


def assembly_rate(p, reps, fused=True):
    F, R, d = p.n_features, p.n_rows, p.dim
    ctx = fls.Context()
    bset = fls.BlockSet(dev_blocks(p), d)
    lda = fls.round_up(R, 4)
    Ab = torch.empty(((F + 1) * lda,), dtype=torch.float64, device="cuda")
    W = torch.empty((F, d), dtype=torch.float64, device="cuda")
    b = torch.empty((F,), dtype=torch.float64, device="cuda")
    s = torch.cuda.Stream()
    ctx.set_stream(s)

    def step():
        if fused:   # one launch for features + prefactors (fls_features_assemble)
            fls.fls_features_assemble(ctx, d, F, p.sigma, p.seed, bset, W=W, b=b, A=Ab, lda=lda)
        else:
            fls.fls_features(ctx, d, F, p.sigma, p.seed, W, b)
            fls.fls_assemble(ctx, W, b, bset, A=Ab, lda=lda)

    with torch.cuda.stream(s):
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        # single-shot latency (host call -> kernels done)
        t0 = time.perf_counter()
        step()
        torch.cuda.synchronize()
        single_ms = 1e3 * (time.perf_counter() - t0)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            step()
        torch.cuda.synchronize()
        for _ in range(3):
            g.replay()
        clk = ClockSampler(0)
        clk.start()
        time.sleep(0.3)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        clk.mark_begin()
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
        torch.cuda.synchronize()
        clk.mark_end()
        clocks = clk.stop()
    fls.fls_sync(ctx)
    ms = e0.elapsed_time(e1) / reps
    ctx.close()
    del Ab
    torch.cuda.empty_cache()
    return ms, single_ms, clocks


def oracle_rate(p, n_rows=64):
    W, b = p.parity_features()
    rows = np.linspace(0, p.n_rows - 1, n_rows).astype(np.int64)
    t0 = time.perf_counter()
    oracle.assemble(W, b, p.blocks, rows=rows, want_scale=False)
    dt = time.perf_counter() - t0
    return n_rows * p.n_features / dt


def main(names):
    hbm_peak, _ = _peaks()
    for name in names:
        p = wl.make_problem(name, "full")
        F, R = p.n_features, p.n_rows
        reps = max(5, min(2000, int(2e10 / (R * F))))
        ms, single_ms, clocks = assembly_rate(p, reps)
        ms_sep, single_sep, _ = assembly_rate(p, reps, fused=False)
        rec = {"config": name, "rows": R, "features": F, "entries": R * F,
               "graph_ms_per_step": ms, "entries_per_s": R * F / (ms / 1e3),
               "hbm_write_gbs": 8.0 * R * (F + 1) / (ms / 1e3) / 1e9,
               "frac_of_copy_peak": 8.0 * R * F / (ms / 1e3) / 1e9 / hbm_peak,
               "single_shot_ms": single_ms, "reps": reps, "clocks": clocks,
               "unfused": {"graph_ms_per_step": ms_sep, "single_shot_ms": single_sep}}
        # end-to-end solve (C5: 262,144-row subset) and fitted-u parity
        import bench

        class Args:
            workload = name
        sol = bench.solve_measure(Args, 1, 0, 0)
        rec["solve"] = sol
        rec["oracle_entries_per_s_all_threads"] = oracle_rate(p)
        rec["oracle_threads"] = oracle.max_threads()
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or wl.CONFIG_NAMES)
