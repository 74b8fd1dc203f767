"""Probe (timing prototype, torch ops): blocked Householder QR = cuSOLVER geqrf on nb-wide panels +
compact-WY trailing updates on cuBLAS DGEMM, vs one monolithic geqrf.  Decides whether libfls's
fls_solve should block the factorisation itself."""
import json
import sys

import torch


def blocked_qr_(A, nb):
    m, n = A.shape
    k = min(m, n)
    taus = []
    for j in range(0, k, nb):
        w = min(nb, k - j)
        a, tau = torch.geqrf(A[j:, j:j + w])
        A[j:, j:j + w] = a
        taus.append(tau)
        if j + w < n:
            V = torch.tril(a, -1)
            V.diagonal().fill_(1.0)
            S = V.T @ V
            # T = (diag(1/tau) + striu(S))^-1  (tau != 0 on random inputs; prototype only)
            Tinv = torch.triu(S, 1) + torch.diag(1.0 / tau)
            T = torch.linalg.solve_triangular(Tinv, torch.eye(w, dtype=A.dtype, device=A.device), upper=True)
            C = A[j:, j + w:]
            Wm = T.T @ (V.T @ C)
            C -= V @ Wm
    return A, torch.cat(taus)


def t_op(fn, reps=2):
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
torch.manual_seed(0)
# correctness on a small case: |diag R| equal to monolithic geqrf's
A0 = torch.randn(3000, 700, dtype=torch.float64, device="cuda")
r_ref = torch.geqrf(A0.clone())[0].diagonal().abs()
r_blk = blocked_qr_(A0.clone(), 64)[0].diagonal().abs()
out["check_rel_diag_err"] = float(((r_ref - r_blk).abs() / r_ref).max())
sizes = [(25000, 4001), (65000, 8001), (262144, 8193)]
for (m, n) in sizes:
    A = torch.randn(m, n, dtype=torch.float64, device="cuda")
    flops = 2 * m * n * n - 2 * n ** 3 / 3
    B = A.clone()
    ms = t_op(lambda: torch.geqrf(B), reps=1)
    out[f"geqrf {m}x{n}"] = {"ms": ms, "tflops": flops / ms / 1e9}
    for nb in (64, 128, 256, 512):
        ms = t_op(lambda: blocked_qr_(B.copy_(A), nb), reps=1)
        out[f"blocked nb={nb} {m}x{n}"] = {"ms": ms, "tflops": flops / ms / 1e9}
    del A, B
    torch.cuda.empty_cache()
    print(json.dumps(out), flush=True)
