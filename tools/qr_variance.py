"""Run-to-run variance of one blocked QR (C4 shape, 10 calls) and per-kernel duration spread
(torch.profiler): python tools/qr_variance.py"""
import sys, os, json, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_10541_b200 import fls
from torch.profiler import profile, ProfilerActivity
m, n = 65000, 8001
lda = (m + 3) // 4 * 4
ctx = fls.Context()
A = torch.randn((n, lda), dtype=torch.float64, device="cuda")
M = torch.empty_like(A)
ts = []
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for it in range(10):
        M.copy_(A)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.profiler.record_function(f"run{it}"):
            e0.record()
            fls.fls_geqrf(ctx, M.view(-1), m, lda, n)
            e1.record()
            torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
print("times", [round(t) for t in ts])
evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
# per-kernel max / median durations
by = {}
for e in evs:
    by.setdefault(e.name[:60], []).append(e.device_time)
for k, v in sorted(by.items(), key=lambda x: -sum(x[1]))[:8]:
    v = sorted(v)
    print(f"{k:60s} n={len(v):5d} sum={sum(v)/1e3:8.1f}ms med={v[len(v)//2]:9.1f}us max={v[-1]:10.1f}us")
