"""Probe: cuBLAS DGEMM rate at the shapes a recursive blocked Householder QR would issue, vs the
cuSOLVER geqrf rate libfls uses today (through torch.geqrf, same library)."""
import json
import time

import torch


def t_op(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {}
for (m, n, k) in [(2000, 2000, 25000), (4000, 4000, 65000), (4096, 4096, 262144), (1024, 4096, 262144),
                  (256, 4096, 262144), (64, 4096, 262144), (8192, 8192, 8192)]:
    A = torch.randn(k, m, dtype=torch.float64, device="cuda")
    B = torch.randn(k, n, dtype=torch.float64, device="cuda")
    ms = t_op(lambda: A.T @ B)
    out[f"AtB {m}x{n}x{k}"] = {"ms": ms, "tflops": 2 * m * n * k / ms / 1e9}
    del A, B
for (m, n) in [(25000, 4001), (65000, 8001)]:
    A = torch.randn(m, n, dtype=torch.float64, device="cuda")
    ms = t_op(lambda: torch.geqrf(A), reps=2)
    out[f"geqrf {m}x{n}"] = {"ms": ms, "tflops": (2 * m * n * n - 2 * n ** 3 / 3) / ms / 1e9}
    del A
print(json.dumps(out, indent=1))
