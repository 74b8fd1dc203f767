"""Interleaved A/B of the assembly launch plan's guided tail (FLS_TAIL_PCT / FLS_TAIL_FPC, read
per call by asm_plan) on the bench's call (fls_features_assemble, 10-step CUDA graphs), with a
bit-identity check of [A | b] against the first setting.

    python tools/ab_tail.py --configs c2_poisson2d c3_poisson5d --settings 0:4 10:4 20:2 --rounds 3

A setting is PCT:FPC (PCT = 0: no tail).  Prints one line per (round, config, setting) and a
median summary.
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as wl  # noqa: E402
from paper_2602_10541_b200 import fls  # noqa: E402


def graph_us(fn, s, per_graph, min_ms):
    with torch.cuda.stream(s):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(per_graph):
                fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.replay()
        e1.record(s)
        torch.cuda.synchronize()
        one = e0.elapsed_time(e1)
        reps = max(3, int(min_ms / max(one, 1e-3)))
        e0.record(s)
        for _ in range(reps):
            g.replay()
        e1.record(s)
        torch.cuda.synchronize()
    return 1e3 * e0.elapsed_time(e1) / (reps * per_graph)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["c2_poisson2d"])
    ap.add_argument("--settings", nargs="+", default=["0:4", "10:4", "20:4"])
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--min-ms", type=float, default=40.0)
    ap.add_argument("--env", default="FLS_TAIL_PCT:FLS_TAIL_FPC",
                    help="the two variables a setting A:B assigns")
    a = ap.parse_args()
    v1, v2 = a.env.split(":")
    s = torch.cuda.Stream()
    probs = {}
    for name in a.configs:
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
        fn = (lambda ctx=ctx, d=d, F=F, p=p, bset=bset, W=W, b=b, Ab=Ab, lda=lda:
              fls.fls_features_assemble(ctx, d, F, p.sigma, p.seed, bset, W=W, b=b, A=Ab, lda=lda))
        per_graph = 10 if p.n_rows * F <= 2e8 else 1
        probs[name] = (fn, Ab, W, b, per_graph, ctx, F, R, lda)
    ref = {}
    res = {}
    for r in range(a.rounds):
        for name in a.configs:
            fn, Ab, W, b, per_graph, ctx, F, R, lda = probs[name]
            for st in a.settings:
                x1, x2 = st.split(":")
                os.environ[v1], os.environ[v2] = x1, x2
                Ab.fill_(float("nan"))
                fn()
                fls.fls_sync(ctx)
                key = (name, st)
                M = Ab.view(F + 1, lda)[:, :R]  # the padding rows lda > R are never written
                if F * R > 2e9:  # too large to clone: every 97th column, bit for bit
                    M = M[::97].clone()
                if name not in ref:
                    ref[name] = (M.clone(), W.clone(), b.clone())
                same = (torch.equal(M, ref[name][0]) and torch.equal(W, ref[name][1])
                        and torch.equal(b, ref[name][2]))
                del M
                us = graph_us(fn, s, per_graph, a.min_ms)
                res.setdefault(key, []).append(us)
                print(json.dumps({"round": r, "config": name, "setting": st, "us": round(us, 3),
                                  "bit_identical": same}), flush=True)
    for (name, st), v in res.items():
        print("summary", name, st, "median %.3f us" % statistics.median(v), "all", [round(x, 2) for x in v])


if __name__ == "__main__":
    main()
