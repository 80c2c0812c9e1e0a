"""Config 4: one training step of a depth-4 MLP of SVD layers on the GPU vs
the same step composed from the f64 oracle (svd_fwd_bwd + svd_step +
clamp_sigma of oracle/fasth_oracle.c, i.e. svd_layer.hpp:106-202), with the
leaky-ReLU and log|det| regulariser glue restated in numpy."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def oracle_step(layers, x, target, cfg, oracle=None):
    from oracle.oracle import Port
    P = oracle if oracle is not None else Port()
    pre, hs = [], [x]
    h = x
    for k, (U, V, s) in enumerate(layers):
        y = P.svd_fwd_bwd(U, V, s, h, None, cfg.block_width)
        pre.append(y)
        h = np.where(y > 0, y, cfg.slope * y) if k < cfg.depth - 1 else y
        hs.append(h)
    r = h - target
    loss = 0.5 * np.sum(r * r) - cfg.lam * sum(np.sum(np.log(np.abs(s))) for _, _, s in layers)
    grad = r
    new = [None] * cfg.depth
    for k in reversed(range(cfg.depth)):
        U, V, s = layers[k]
        if k < cfg.depth - 1:
            grad = grad * np.where(pre[k] > 0, 1.0, cfg.slope)
        Y, dX, dU, dV, ds = P.svd_fwd_bwd(U, V, s, hs[k], grad, cfg.block_width)
        ds = ds - cfg.lam / s
        new[k] = P.svd_step(U, V, s, dU, dV, ds, cfg.eta, cfg.clamp_eps)
        grad = dX
    return new, loss


def test_mlp_train_step_matches_oracle():
    import torch

    from oracle.oracle import relative_error
    from paper_2009_13977_b200 import mlp

    cfg = mlp.MLPConfig(d=96, depth=4, block_width=16, eta=1e-2, lam=1e-2)
    layers = mlp.random_layers(cfg, seed=3)
    host = [(p.U.double().cpu().numpy(), p.V.double().cpu().numpy(), p.sigma.double().cpu().numpy())
            for p in layers]
    rng = np.random.default_rng(4)
    x = rng.standard_normal((cfg.d, 8))
    target = rng.standard_normal((cfg.d, 8))
    want, want_loss = oracle_step(host, x, target, cfg)
    loss = mlp.train_step(layers, torch.tensor(x, dtype=torch.float32, device="cuda"),
                          torch.tensor(target, dtype=torch.float32, device="cuda"), cfg)
    assert abs(float(loss) - want_loss) <= 1e-4 * abs(want_loss)
    for p, (U, V, s) in zip(layers, want):
        assert relative_error(p.U.double().cpu().numpy(), U) <= 1e-4
        assert relative_error(p.V.double().cpu().numpy(), V) <= 1e-4
        assert relative_error(p.sigma.double().cpu().numpy(), s) <= 1e-4


def test_mlp_train_step_large_batch_matches_chain_path(monkeypatch):
    """The same training step at a batch that selects the large-batch path
    for every layer leg (plans carry no blocks there) against the chain
    kernels (FASTH_LB=0): loss and updated parameters within tolerance."""
    import torch

    from paper_2009_13977_b200 import mlp

    cfg = mlp.MLPConfig(d=512, depth=2, block_width=32, eta=1e-3, lam=1e-3)
    g = torch.Generator(device="cuda").manual_seed(9)
    x = torch.randn(cfg.d, 1024, device="cuda", generator=g)
    target = torch.randn(cfg.d, 1024, device="cuda", generator=g)
    out = {}
    for lb in ("1", "0"):
        monkeypatch.setenv("FASTH_LB", lb)
        layers = mlp.random_layers(cfg, seed=5)
        loss = float(mlp.train_step(layers, x, target, cfg))
        out[lb] = (loss, layers)
    (l1, a), (l0, b) = out["1"], out["0"]
    assert abs(l1 - l0) <= 1e-4 * abs(l0)
    rel = lambda u, v: float((u.double() - v.double()).norm() / v.double().norm())
    for p, q in zip(a, b):
        assert rel(p.U, q.U) <= 1e-4 and rel(p.V, q.V) <= 1e-4 and rel(p.sigma, q.sigma) <= 1e-4
