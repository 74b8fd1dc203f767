"""Kernel timeline of a small config's steady-state step (where C2's 17.5 us goes).

Captures a graph of N consecutive fls_features_assemble calls (the bench's call), replays it under
torch.profiler (CUPTI kernel records carry device start / end timestamps also inside graphs) and
prints, per step, each kernel's duration and the gaps between consecutive kernels:

    python tools/step_timeline.py [c2_poisson2d] [--steps 10] [--replays 20]

Output: one JSON line per config with the median over replays of
  step_us      time between the starts of consecutive assembly kernels
  kernels      {name: median duration us}
  gaps         {"<prev> -> <next>": median gap us} (end of one kernel to start of the next)
"""
import argparse
import json
import os
import statistics
import sys
import tempfile

import torch
from torch.profiler import ProfilerActivity, profile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as wl  # noqa: E402
from paper_2602_10541_b200 import fls  # noqa: E402


def short(name):
    if "features_prefactor" in name:
        return "prefactor"
    if "assemble_cm_kernel" in name:
        return "assemble_fused" if "FusedBatch" in name else "assemble"
    return name[:40]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c2_poisson2d"])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--replays", type=int, default=20)
    a = ap.parse_args()
    s = torch.cuda.Stream()
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
        fn = lambda: fls.fls_features_assemble(ctx, d, F, p.sigma, p.seed, bset, W=W, b=b, A=Ab, lda=lda)
        with torch.cuda.stream(s):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(a.steps):
                    fn()
            for _ in range(20):
                g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(200):
                g.replay()
            e1.record(s)
            torch.cuda.synchronize()
            us_step_events = 1e3 * e0.elapsed_time(e1) / (200 * a.steps)
            with profile(activities=[ProfilerActivity.CUDA]) as prof:
                for _ in range(a.replays):
                    g.replay()
                torch.cuda.synchronize()
        with tempfile.NamedTemporaryFile(suffix=".json", delete=False) as tf:
            path = tf.name
        prof.export_chrome_trace(path)
        ev = json.load(open(path))["traceEvents"]
        os.unlink(path)
        ks = sorted([(e["ts"], e["dur"], short(e["name"])) for e in ev
                     if e.get("cat") == "kernel"], key=lambda t: t[0])
        durs, gaps, steps = {}, {}, []
        last_asm = None
        for i, (ts, dur, nm) in enumerate(ks):
            durs.setdefault(nm, []).append(dur)
            if i:
                pts, pdur, pnm = ks[i - 1]
                gaps.setdefault(f"{pnm} -> {nm}", []).append(ts - (pts + pdur))
            if nm.startswith("assemble"):
                if last_asm is not None and ts - last_asm < 1000:
                    steps.append(ts - last_asm)
                last_asm = ts
        med = lambda v: round(statistics.median(v), 3)
        print(json.dumps({"config": name, "us_per_step_events": round(us_step_events, 3),
                          "step_us": med(steps) if steps else None,
                          "kernels": {k: med(v) for k, v in durs.items()},
                          "gaps": {k: med(v) for k, v in gaps.items()},
                          "n_kernels": len(ks)}), flush=True)


if __name__ == "__main__":
    main()
