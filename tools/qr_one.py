"""One blocked QR of an m x n random block (profiling helper): python tools/qr_one.py m n [reps]"""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2602_10541_b200 import fls  # noqa: E402

m, n = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
ctx = fls.Context()
lda = (m + 3) // 4 * 4
A = torch.randn((n, lda), dtype=torch.float64, device="cuda")
M = torch.empty_like(A)
for _ in range(reps):
    M.copy_(A)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fls.fls_geqrf(ctx, M.view(-1), m, lda, n)
    e1.record()
    torch.cuda.synchronize()
    print(f"{m} x {n}: {e0.elapsed_time(e1):.2f} ms")
