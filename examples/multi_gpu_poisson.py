"""Algorithm 1 row-sharded over the GPUs of one node: each rank assembles its rows
of the stacked [A_pde; lambda A_bc | rhs] (no collective), then the least-squares solve runs as
TSQR inside libfls (R factors stored into rank 0's memory over NVLink by CUDA IPC, beta back on
every rank).  2-D Poisson -Lap u = f on [0,1]^2, u* = sin(pi x) sin(2 pi y).

    torchrun --nproc-per-node N examples/multi_gpu_poisson.py      (one rank per GPU)
    python examples/multi_gpu_poisson.py                            (one GPU)

FLS_EXAMPLE_BACKEND=gloo runs the ranks with a host control plane instead of NCCL (e.g. several
processes sharing one GPU for a test)."""
import math
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_10541_b200 import fls, operators as ops  # noqa: E402
from paper_2602_10541_b200.pipeline import solve_linear  # noqa: E402

if "WORLD_SIZE" in os.environ:
    backend = os.environ.get("FLS_EXAMPLE_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
rank = dist.get_rank() if dist.is_initialized() else 0

ctx = fls.Context()
# every rank draws the same points (counter-based, seeded) and assembles only its own rows
Xi = fls.fls_sample_box(ctx, 2, 8000, [0, 0], [1, 1], seed=0, stream=3)
Xb = fls.fls_sample_faces(ctx, 2, 400, [0, 1], [0, 0], [1, 1], seed=0, stream=4)
u_star = lambda X: torch.sin(math.pi * X[:, 0]) * torch.sin(2 * math.pi * X[:, 1])
blocks = [fls.Block(Xi, ops.laplacian(2, -1.0), 1.0, 5 * math.pi ** 2 * u_star(Xi)),
          fls.Block(Xb, ops.identity(2), 100.0, u_star(Xb))]
sol = solve_linear(ctx, dim=2, n_features=2500, sigma=5.0, seed=0, blocks=blocks)
Xt = fls.fls_sample_box(ctx, 2, 10000, [0, 0], [1, 1], seed=0, stream=6)
u = sol.evaluate(Xt)
err = float(torch.linalg.norm(u - u_star(Xt)) / torch.linalg.norm(u_star(Xt)))
world = dist.get_world_size() if dist.is_initialized() else 1
if rank == 0:
    print(f"{world} rank(s): relative L2 error vs u* {err:.2e}, residual {sol.resid_norm:.3e}")
if dist.is_initialized():
    dist.destroy_process_group()
