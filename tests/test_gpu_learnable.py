"""GPU learnable bandwidth (App. E) vs the oracle: the reparameterised features, the outer-loss
gradient dLout/dL (scalar and Cholesky), and a short AdamW trajectory."""
import math

import numpy as np
import pytest
import torch

import oracle.learnable as ol
import workloads as wl
from gpu_common import dev_blocks

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2602_10541_b200 import fls
    from paper_2602_10541_b200.learnable import fit_bandwidth, outer_loss_and_grad


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return fls.Context()


def _setup():
    p = wl.make_helmholtz2d(n_int=300, per_edge=20, n_features=60)
    W_hat, b = p.parity_features()
    return p, W_hat, b


def test_features_transform(ctx):
    g = np.random.default_rng(0)
    Wh = g.normal(size=(1001, 3))
    L = np.tril(g.normal(size=(3, 3))) + 3 * np.eye(3)
    W = fls.fls_features_transform(ctx, L.tolist(), torch.from_numpy(Wh).cuda()).cpu().numpy()
    assert np.allclose(W, Wh @ L.T, rtol=1e-15, atol=1e-14)


@pytest.mark.parametrize("L", [[[5.0, 0.0], [0.0, 5.0]], [[3.0, 0.0], [0.7, 4.0]]])
def test_bandwidth_gradient_matches_oracle(ctx, L):
    p, W_hat, b = _setup()
    loss_o, G_o, _ = ol.outer_grad(np.array(L), W_hat, b, p.blocks)
    loss, G, _ = outer_loss_and_grad(ctx, L, torch.from_numpy(W_hat).cuda(),
                                     torch.from_numpy(b).cuda(), dev_blocks(p))
    G = np.array(G)
    assert abs(loss - loss_o) <= 1e-8 * loss_o
    assert np.abs(G - G_o).max() <= 1e-7 * np.abs(G_o).max(), (G, G_o)


@pytest.mark.parametrize("L", [[[5.0, 0.0], [0.0, 5.0]], [[4.0, 0.0], [0.5, 5.0]]])
def test_bandwidth_gradient_with_coefficient_field_matches_oracle(ctx, L):
    """variable-coefficient Helmholtz (k^2 (1 + x_1) u as a coefficient field)"""
    p = wl.make_helmholtz2d_var(n_int=300, per_edge=20, n_features=60)
    W_hat, b = p.parity_features()
    loss_o, G_o, _ = ol.outer_grad(np.array(L), W_hat, b, p.blocks)
    loss, G, _ = outer_loss_and_grad(ctx, L, torch.from_numpy(W_hat).cuda(),
                                     torch.from_numpy(b).cuda(), dev_blocks(p))
    G = np.array(G)
    assert abs(loss - loss_o) <= 1e-8 * loss_o
    assert np.abs(G - G_o).max() <= 1e-7 * np.abs(G_o).max(), (G, G_o)


def test_adamw_trajectory_matches_oracle(ctx):
    p, W_hat, b = _setup()
    steps, lr = 6, 0.05
    Lg, hist = fit_bandwidth(ctx, torch.from_numpy(W_hat).cuda(), torch.from_numpy(b).cuda(),
                             dev_blocks(p), mode="scalar", init=5.0, steps=steps, lr=lr)
    # oracle side: the same outer loop written out (Adam moments, bias correction, no decay)
    s, m, v = 5.0, 0.0, 0.0
    for t in range(1, steps + 1):
        _, G, _ = ol.outer_grad(s * np.eye(2), W_hat, b, p.blocks)
        g = np.trace(G)
        m = 0.9 * m + 0.1 * g
        v = 0.999 * v + 0.001 * g * g
        s -= lr * (m / (1 - 0.9 ** t)) / (math.sqrt(v / (1 - 0.999 ** t)) + 1e-8)
    assert abs(Lg[0][0] - s) <= 1e-7 * s
    assert hist[-1]["loss"] < hist[0]["loss"]


def test_bandwidth_gradient_with_ridge_matches_oracle(ctx):
    """Tikhonov inner solve (sqrt_mu > 0): the ridge-augmented outer loss and its exact envelope
    gradient (reading B2) vs the oracle, which is pinned to central FD of the same loss"""
    p, W_hat, b = _setup()
    L = [[3.0, 0.0], [0.7, 4.0]]
    sq = 3e-2
    loss_o, G_o, _ = ol.outer_grad(np.array(L), W_hat, b, p.blocks, sqrt_mu=sq)
    loss, G, _ = outer_loss_and_grad(ctx, L, torch.from_numpy(W_hat).cuda(),
                                     torch.from_numpy(b).cuda(), dev_blocks(p), sqrt_mu=sq)
    G = np.array(G)
    assert abs(loss - loss_o) <= 1e-8 * loss_o
    assert np.abs(G - G_o).max() <= 1e-7 * np.abs(G_o).max(), (G, G_o)
