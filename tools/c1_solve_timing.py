"""fls_solve on the full C1 system, 6 calls (first-call vs steady-state latency)."""
import sys, time, torch
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import workloads as wl
from paper_2602_10541_b200 import fls
p = wl.make_problem("c1_poisson1d", "full")
W, b = p.parity_features()
ctx = fls.Context()
blocks = [fls.Block(torch.from_numpy(x.X).cuda(), x.terms, x.weight, torch.from_numpy(x.values).cuda()) for x in p.blocks]
Wd, bd = torch.from_numpy(W).cuda(), torch.from_numpy(b).cuda()
F, R = p.n_features, p.n_rows
for it in range(6):
    Ab, lda = fls.fls_assemble(ctx, Wd, bd, blocks)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    beta, res = fls.fls_solve(ctx, Ab, R, lda, F)
    torch.cuda.synchronize()
    print(it, round((time.perf_counter() - t0) * 1e3, 2), "ms")
