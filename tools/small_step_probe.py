"""Where a small config's step goes (C1/C2 are launch-latency bound).

For each config: the graph-replayed step (fused features + assembly, what bench.py's
per_config reports), the same with fixed W, b (prefactor + assembly launches), kernel
durations from torch.profiler, and a floor: a graph of two empty-ish torch kernels.

    python tools/small_step_probe.py [c1_poisson1d c2_poisson2d ...]
"""
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as wl  # noqa: E402
from paper_2602_10541_b200 import fls  # noqa: E402


def graph_us(fn, s, reps=2000, per_graph=1):
    """us per step: a graph of per_graph steps replayed reps / per_graph times"""
    reps = max(1, reps // per_graph)
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(per_graph):
                fn()
        for _ in range(10):
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
        torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / (reps * per_graph)


def main(names):
    s = torch.cuda.Stream()
    x = torch.zeros(1, device="cuda")
    floor2 = graph_us(lambda: (x.add_(1), x.add_(1)), s)
    floor1 = graph_us(lambda: x.add_(1), s)
    for name in names:
        p = wl.make_problem(name, "full")
        F, R, d = p.n_features, p.n_rows, p.dim
        ctx = fls.Context(stream=s)
        bset = fls.BlockSet([fls.Block(torch.from_numpy(b.X).cuda(), b.terms, b.weight,
                                       torch.from_numpy(b.values).cuda(),
                                       torch.from_numpy(b.fields).cuda() if b.fields is not None else None)
                             for b in p.blocks], d)
        lda = fls.round_up(R, 4)
        Ab = torch.empty(((F + 1) * lda,), dtype=torch.float64, device="cuda")
        W = torch.empty((F, d), dtype=torch.float64, device="cuda")
        b = torch.empty((F,), dtype=torch.float64, device="cuda")
        fused = lambda: fls.fls_features_assemble(ctx, d, F, p.sigma, p.seed, bset, W=W, b=b, A=Ab, lda=lda)
        fused()
        sep = lambda: fls.fls_assemble(ctx, W, b, bset, A=Ab, lda=lda)
        t_fused = graph_us(fused, s)
        t_sep = graph_us(sep, s)
        t_fused10 = graph_us(fused, s, per_graph=10)
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            with torch.cuda.stream(s):
                for _ in range(50):
                    fused()
            torch.cuda.synchronize()
        kern = {}
        for ev in prof.key_averages():
            if ev.device_type.name == "CUDA" and ev.count >= 50:
                kern[ev.key[:60]] = round(ev.device_time_total / ev.count, 2)
        print(json.dumps({"config": name, "graph_us_fused_step": t_fused,
                          "graph10_us_fused_step": t_fused10,
                          "graph_us_prefactor_plus_assembly": t_sep,
                          "kernel_us": kern, "floor_graph_us_1_kernel": floor1,
                          "floor_graph_us_2_kernels": floor2,
                          "hbm_time_us_at_copy_peak": 8 * R * (F + 1) / 6458.7e9 * 1e6}), flush=True)
        ctx.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1_poisson1d", "c2_poisson2d", "c3_poisson5d"])
