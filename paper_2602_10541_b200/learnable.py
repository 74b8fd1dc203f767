"""Learnable-bandwidth Fast-LSQ (App. E, Alg. 2) on the device.

    W_j = L W^_j  (scalar: L = sigma I;  anisotropic: lower-triangular Cholesky factor)
    beta* = argmin ||A(L) beta - b||^2            (inner exact solve, fls_solve)
    Lout  = ||A(L) beta* - b||^2                  (outer loss)
    dLout/dL via fls_bandwidth_grad (no differentiation through the solve: beta* is optimal;
    with a ridge the loss gains mu ||beta*||^2 so that this stays exact, reading B2)
    AdamW on the d(d+1)/2 (or 1) bandwidth parameters

Every arithmetic step on F- or R-sized data is a libfls call; the optimiser updates the
handful of bandwidth scalars on the host.  AdamW hyperparameters are not given in the paper
(reading B1 in DESIGN.md): lr, betas (0.9, 0.999), eps 1e-8, weight decay 0 by default.
"""
from __future__ import annotations

import math
from typing import List, Sequence

import torch

from . import fls


def outer_loss_and_grad(ctx, L, W_hat, b, blocks: Sequence[fls.Block], sqrt_mu: float = 0.0,
                        normalize: bool = True):
    """(Lout, dLout/dL (d x d), beta) at the factor L.  With sqrt_mu > 0 the loss is the
    ridge-augmented Lout + mu ||beta*||^2 -- the objective the inner solve minimises -- whose
    gradient the envelope formula gives exactly (reading B2); at mu = 0 it is Lout."""
    F, d = int(W_hat.shape[0]), int(W_hat.shape[1])
    W = fls.fls_features_transform(ctx, L, W_hat)
    R = sum(blk.n for blk in blocks)
    extra = F if sqrt_mu > 0 else 0
    Ab, lda = fls.fls_assemble(ctx, W, b, blocks, normalize=normalize, extra_rows=extra)
    beta, _ = fls.fls_solve_mu(ctx, Ab, R, lda, F, sqrt_mu)
    loss = 0.0
    rblocks = []
    for blk in blocks:
        Abeta = fls.fls_eval_block(ctx, W, b, beta, blk, normalize=normalize)   # w L[u_N](x_i)
        vals = blk.values if blk.values is not None else torch.zeros_like(Abeta)
        r = fls.fls_axpy(ctx, -blk.weight, vals, Abeta)                        # w (L[u] - v)
        loss += fls.fls_frob2(ctx, r, r.numel(), max(r.numel(), 1), 1) if r.numel() else 0.0
        rblocks.append(fls.Block(blk.X, blk.terms, blk.weight, r, blk.fields))
    if sqrt_mu > 0:
        loss += sqrt_mu * sqrt_mu * fls.fls_frob2(ctx, beta, F, F, 1)
    G = fls.fls_bandwidth_grad(ctx, W, W_hat, b, rblocks, beta, normalize=normalize)
    return loss, G, beta


class AdamW:
    """Loshchilov & Hutter's decoupled-weight-decay Adam on a list of floats"""

    def __init__(self, params, lr=0.05, betas=(0.9, 0.999), eps=1e-8, weight_decay=0.0):
        self.p = [float(v) for v in params]
        self.lr, self.b1, self.b2, self.eps, self.wd = lr, betas[0], betas[1], eps, weight_decay
        self.m = [0.0] * len(self.p)
        self.v = [0.0] * len(self.p)
        self.t = 0

    def step(self, grads):
        self.t += 1
        for i, g in enumerate(grads):
            self.m[i] = self.b1 * self.m[i] + (1 - self.b1) * g
            self.v[i] = self.b2 * self.v[i] + (1 - self.b2) * g * g
            mh = self.m[i] / (1 - self.b1 ** self.t)
            vh = self.v[i] / (1 - self.b2 ** self.t)
            self.p[i] -= self.lr * (mh / (math.sqrt(vh) + self.eps) + self.wd * self.p[i])
        return self.p


def _L_from(params, d, mode):
    if mode == "scalar":
        return [[params[0] if k == l else 0.0 for l in range(d)] for k in range(d)]
    L = [[0.0] * d for _ in range(d)]
    it = iter(params)
    for k in range(d):
        for l in range(k + 1):
            L[k][l] = next(it)
    return L


def _grad_params(G, d, mode):
    if mode == "scalar":
        return [sum(G[k][k] for k in range(d))]
    return [G[k][l] for k in range(d) for l in range(k + 1)]


def fit_bandwidth(ctx, W_hat, b, blocks, *, mode: str = "scalar", init=1.0, steps: int = 80,
                  lr: float = 0.05, weight_decay: float = 0.0, sqrt_mu: float = 0.0):
    """Alg. 2.  mode 'scalar' learns sigma (init: float), 'cholesky' the
    lower-triangular L (init: d x d list, or a float for init * I).  Returns (L, history)."""
    d = int(W_hat.shape[1])
    if mode == "scalar":
        params = [float(init)]
    else:
        L0 = init if isinstance(init, (list, tuple)) else [[init if k == l else 0.0 for l in range(d)]
                                                           for k in range(d)]
        params = [L0[k][l] for k in range(d) for l in range(k + 1)]
    opt = AdamW(params, lr=lr, weight_decay=weight_decay)
    hist: List[dict] = []
    for _ in range(steps):
        L = _L_from(opt.p, d, mode)
        loss, G, _ = outer_loss_and_grad(ctx, L, W_hat, b, blocks, sqrt_mu)
        g = _grad_params(G, d, mode)
        hist.append({"loss": loss, "params": list(opt.p), "grad": g})
        opt.step(g)
    return _L_from(opt.p, d, mode), hist
