"""Newton-Fast-LSQ on a nonlinear PDE: -Lap u + u^3 = f on [0,1]^2, u = g on the
boundary, u* = sin(pi x) sin(pi y).  Points sampled on the device, features drawn on the device,
each Newton step one Tikhonov least-squares solve (mu = 1e-10) of the analytically assembled
Jacobian.  Run on a GPU:  python examples/nonlinear_poisson.py"""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_10541_b200 import fls, operators as ops  # noqa: E402
from paper_2602_10541_b200.newton import solve_nonlinear  # noqa: E402

ctx = fls.Context()
Xi = fls.fls_sample_box(ctx, 2, 5000, [0, 0], [1, 1], seed=0, stream=3)              # interior
Xb = fls.fls_sample_faces(ctx, 2, 200, [0, 1], [0, 0], [1, 1], seed=0, stream=4)      # 4 edges
u_star = lambda X: torch.sin(math.pi * X[:, 0]) * torch.sin(math.pi * X[:, 1])
f = 2 * math.pi ** 2 * u_star(Xi) + u_star(Xi) ** 3
pde = fls.Block(Xi, ops.laplacian(2, -1.0), 1.0, f)                 # L u = -Lap u
bc = fls.Block(Xb, ops.identity(2), 100.0, u_star(Xb))              # lambda u = lambda g
W, b = fls.fls_features(ctx, 2, 1500, 3.0, seed=0)
beta, hist = solve_nonlinear(ctx, W, b, pde, [bc], "poly", [0.0, 0.0, 0.0, 1.0], max_iter=10)
Xt = fls.fls_sample_box(ctx, 2, 10000, [0, 0], [1, 1], seed=0, stream=6)
u = fls.fls_eval(ctx, W, b, beta, Xt)
err = float(torch.linalg.norm(u - u_star(Xt)) / torch.linalg.norm(u_star(Xt)))
print(f"{len(hist) - 1} Newton iterations, relative L2 error vs u*: {err:.2e}")
