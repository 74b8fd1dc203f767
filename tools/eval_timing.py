"""fls_eval timing at the C5 solve shape (10,000 points x 8,192 features): u_N (sin-only path) vs a mixed-parity operator."""
import sys, torch
sys.path.insert(0, ".")
from paper_2602_10541_b200 import fls
ctx = fls.Context()
F, d = 8192, 3
W, b = fls.fls_features(ctx, d, F, 3.0, 0)
beta = torch.randn(F, dtype=torch.float64, device="cuda")
X = torch.rand((10000, d), dtype=torch.float64, device="cuda")
for terms, nm in ((None, "u (sin only)"), ([((1, 0, 0), 1.0, -1), ((2, 0, 0), 1.0, -1)], "mixed (sin+cos)")):
    for _ in range(3): fls.fls_eval(ctx, W, b, beta, X, terms=terms)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): fls.fls_eval(ctx, W, b, beta, X, terms=terms)
    e1.record(); torch.cuda.synchronize()
    print(nm, round(e0.elapsed_time(e1) / 20, 4), "ms")
