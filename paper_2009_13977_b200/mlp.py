"""Depth-L MLP of SVD-reparameterised layers (BASELINE config 4).

The reference's training template is demos/svd_layer_demo.cpp:25-43 (one
layer: forward, residual loss, svd_backward, svd_step, clamp_sigma).  Config
4 stacks L = 4 such layers at d = 784 with an invertible leaky-ReLU between
them and a log|det W| regulariser per layer, so every step exercises the
Sigma-side ops:

    h_0 = x;   h_{k+1} = leaky(W_k h_k) (k < L-1);   y = W_{L-1} h_{L-1}
    loss = 1/2 ||y - target||^2  -  lam * sum_k log|det W_k|

with W_k = U_k Sigma_k V_k^T.  d log|det W| / d sigma_i = 1 / sigma_i
(matops.hpp:57-66), so the regulariser enters dSigma in closed form.  All
chain work (both legs of every layer, forward and backward) and the
step/clamp run in the library's sm_100a kernels; the activation, the loss
and the regulariser's log|sigma| sum and -lam/sigma term are elementwise
torch ops on the same stream (fb.log_abs_det is the library's kernel for
log|det| but returns a host scalar, which would synchronise the step).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import fasth as fb


@dataclass
class MLPConfig:
    d: int = 784
    depth: int = 4
    block_width: int = 32
    slope: float = 0.1       # leaky-ReLU negative slope
    lam: float = 1e-3        # log|det| regulariser weight
    eta: float = 1e-3        # SGD step (svd_layer.hpp:158)
    clamp_eps: float = 0.5   # clamp_sigma epsilon (svd_layer.hpp:196)
    prebuild: bool = True    # build layer k+1's WY blocks while layer k sweeps (svd_plan)


def random_layers(cfg: MLPConfig, seed: int = 0, device="cuda"):
    """SvdParam::random-like init (svd_layer.hpp:46-71): unit Gaussian
    vectors normalised, sigma ~ U(0.5, 2) as bench.hpp:129-131."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    layers = []
    for _ in range(cfg.depth):
        U = torch.randn(cfg.d, cfg.d, generator=g)
        V = torch.randn(cfg.d, cfg.d, generator=g)
        U /= U.norm(dim=1, keepdim=True)
        V /= V.norm(dim=1, keepdim=True)
        s = torch.rand(cfg.d, generator=g) * 1.5 + 0.5
        layers.append(fb.SvdParam(cfg.d, cfg.d, U.to(device), V.to(device), s.to(device)))
    return layers


def train_step(layers, x, target, cfg: MLPConfig, ctx=None):
    """One full fwd + bwd + SGD step; updates `layers` in place and returns
    the loss as a 0-d device tensor (no host sync)."""
    hs, pre, tapes = [x], [], []
    h = x
    m = x.shape[1]
    # layer k+1's WY blocks are built on the side stream while layer k sweeps
    # (they depend only on that layer's U and V)
    plan = fb.svd_plan(layers[0], m, cfg.block_width, ctx=ctx) if cfg.prebuild else None
    for k, p in enumerate(layers):
        nxt = (fb.svd_plan(layers[k + 1], m, cfg.block_width, ctx=ctx)
               if cfg.prebuild and k + 1 < len(layers) else None)
        y, tape = fb.svd_forward(p, h, cfg.block_width, ctx=ctx, plan=plan)
        plan = nxt
        tapes.append(tape)
        pre.append(y)
        h = torch.nn.functional.leaky_relu(y, cfg.slope) if k < cfg.depth - 1 else y
        hs.append(h)
    r = h - target
    logdet = torch.stack([torch.log(p.sigma.abs()).sum() for p in layers]).sum()
    loss = 0.5 * (r * r).sum() - cfg.lam * logdet
    grad = r
    for k in reversed(range(cfg.depth)):
        p = layers[k]
        if k < cfg.depth - 1:
            grad = grad * torch.where(pre[k] > 0, 1.0, cfg.slope)
        g = fb.svd_backward(p, tapes[k], grad)
        # regulariser: d(-lam log|det W|)/d sigma = -lam / sigma
        g.grad_sigma.sub_(cfg.lam / p.sigma)
        grad = g.grad_input
        fb.svd_step(p, g, cfg.eta, clamp_epsilon=cfg.clamp_eps, inplace=True, ctx=ctx)
    return loss


def flops_per_step(cfg: MLPConfig, m: int) -> float:
    """each layer = 2 FastH fwd+bwd = 2 (12 d n m + 4 d n b)."""
    d = cfg.d
    return cfg.depth * 2 * (12.0 * d * d * m + 4.0 * d * d * cfg.block_width)
