"""leaf-kernel time of one blocked QR (torch.profiler): python tools/leaf_time.py m n"""
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2602_10541_b200 import fls  # noqa: E402

m, n = int(sys.argv[1]), int(sys.argv[2])
ctx = fls.Context()
lda = (m + 3) // 4 * 4
A = torch.randn((n, lda), dtype=torch.float64, device="cuda")
M = A.clone()
fls.fls_geqrf(ctx, M.view(-1), m, lda, n)
M.copy_(A)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    fls.fls_geqrf(ctx, M.view(-1), m, lda, n)
    torch.cuda.synchronize()
for e in prof.key_averages():
    if "qr_leaf" in e.key:
        print(f"{e.key[:40]} calls {e.count} total {e.device_time_total / 1e3:.2f} ms avg {e.device_time_total / e.count:.1f} us")
