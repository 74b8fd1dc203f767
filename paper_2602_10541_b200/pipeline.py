"""Algorithm 1 end to end on the device -- the call a user makes.

    sol = solve_linear(ctx, dim=2, n_features=2000, sigma=5.0, seed=0, blocks=[pde, bc])
    u = sol.evaluate(X_test)               # u_N at new points (fls_eval)
    r = sol.evaluate(X_test, terms=L)      # L[u_N] (PDE residual check)

Steps: fls_features (line 1) -> caller's collocation blocks (line 2, e.g. fls_sample_box /
fls_sample_faces) -> fls_assemble (lines 3-5; lines 1 + 3-5 as fls_features_assemble for a single
bandwidth) -> fls_solve / TSQR over the process group
(line 5) -> u_N (line 6).  Row sharding when torch.distributed is initialised: each rank
assembles its own rows [floor(r R/P), floor((r+1) R/P)) of the stacked blocks; no data-path
collective until the TSQR gather.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional, Sequence

import torch
import torch.distributed as dist

from . import fls
from .dist import shard_range, tsqr_solve


@dataclasses.dataclass
class Solution:
    ctx: fls.Context
    W: torch.Tensor
    b: torch.Tensor
    beta: torch.Tensor
    resid_norm: float
    normalize: bool = True

    def evaluate(self, X: torch.Tensor, terms: Optional[Sequence] = None) -> torch.Tensor:
        return fls.fls_eval(self.ctx, self.W, self.b, self.beta, X, terms=terms,
                            normalize=self.normalize)


def solve_linear(ctx: fls.Context, *, dim: int, n_features: int, sigma, seed: int,
                 blocks: List[fls.Block], ridge_rel: float = 0.0, normalize: bool = True,
                 block_features: Optional[Sequence[int]] = None) -> Solution:
    """sigma: a float, or a list of per-block bandwidths with block_features.
    ridge_rel: tau of sqrt(mu) = tau ||A||_F (Tikhonov; reading A16).
    blocks hold ALL rows on every rank (the points are small); each rank assembles its shard."""
    R = sum(blk.n for blk in blocks)
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    a, e = shard_range(R, rank, world)
    n_local = e - a
    if block_features is not None:
        W, b = fls.fls_features_blocks(ctx, dim, block_features, sigma, seed)
        F = int(W.shape[0])
        extra = F if (ridge_rel > 0 and world == 1) else 0
        Ab, lda = fls.fls_assemble(ctx, W, b, blocks, normalize=normalize, row_begin=a, row_end=e,
                                   extra_rows=extra)
    else:   # one bandwidth: features + prefactors fused into one launch (fls_features_assemble)
        F = int(n_features)
        extra = F if (ridge_rel > 0 and world == 1) else 0
        W, b, Ab, lda = fls.fls_features_assemble(ctx, dim, F, float(sigma), seed, blocks,
                                                  normalize=normalize, row_begin=a, row_end=e,
                                                  extra_rows=extra)
    beta, res = tsqr_solve(Ab, n_local, lda, F, ridge_rel=ridge_rel, ctx=ctx)
    return Solution(ctx, W, b, beta, res, normalize)
