"""Every BASELINE.json config pinned to the reference oracle on the GPU.

The oracle is ``oracle/_ref`` (the unmodified reference headers compiled
here, ``Ref``) wherever it is present, else the C restatement (``Port``).
Inputs come from the reference's own seeded generators (bench.hpp:117-134)
where the shape is one the reference benchmark draws, so the GPU sees the
reference's exact inputs.  Each test records its measured error per output
(printed; also appended as JSON lines to ``$FASTH_PARITY_LOG`` when set).

Tolerance (north_star): relative error
||a - b||_F / max(||b||_F, 1) (matrix.hpp:106-110) <= 1e-4 on UX, dX, dV.

configs (BASELINE.json):
  [0] d=64, b=8, m=32 ............ tests/test_gpu_fasth.py goldens ("cfg1")
  [1] d=784, b=32, m=32 .......... tests/test_gpu_fasth.py::test_cfg2_metric_config_vs_reference
                                   + here as the SVD layer
  [2] d sweep 256..4096, b 32/64 . here: mul, exp, Cayley at d in {3072, 4096}
  [3] depth-4 MLP at d=784 ....... here
  [4] d=2048, batch 8192/GPU ..... here: UX, dX, dV over the full batch,
                                   against the reference
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-4


def _oracle():
    from oracle.oracle import Port, Ref
    try:
        return Ref()
    except Exception:
        return Port()


@pytest.fixture(scope="module")
def fb():
    import torch
    from paper_2009_13977_b200 import fasth
    assert torch.cuda.is_available()
    return fasth


@pytest.fixture(scope="module")
def ref():
    return _oracle()


def dev(a):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def host(t):
    return t.detach().double().cpu().numpy()


def rel(a, b):
    from oracle.oracle import relative_error
    return relative_error(host(a) if not isinstance(a, np.ndarray) else a, b)


def record(config, **errs):
    rec = {"config": config, **{k: float(v) for k, v in errs.items()}}
    print("PARITY", json.dumps(rec))
    path = os.environ.get("FASTH_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")
    return rec


# ---- config [2]: the d sweep at its largest sizes ----------------------------

@pytest.mark.parametrize("d", [3072, 4096])
@pytest.mark.parametrize("b", [32, 64])
def test_config3_mul_large_d_vs_reference(fb, ref, d, b):
    """op=mul (bench.hpp:117-121 generator, seed 0) at batch 32: the chain
    kernels with 16-wide internal blocks (capi.cpp internal_b)."""
    V, X, G = ref.gen_mul(0, d, 32) if hasattr(ref, "gen_mul") else (
        np.random.default_rng(d).standard_normal((d, d)),) + tuple(
        np.random.default_rng(d + 1).standard_normal((2, d, 32)))
    want = ref.fasth_fwd_bwd(V, X, G, b)
    got = fb.fasth_forward_backward(dev(V), dev(X), dev(G), b)
    got = (got[0], got[1].grad_input, got[1].grad_vectors)
    tape = fb.fasth_forward(dev(V), dev(X), b)
    back = fb.fasth_backward(tape, dev(G))
    two = (tape.output(), back.grad_input, back.grad_vectors)
    e = [rel(a, w) for a, w in zip(got, want)]
    e2 = [rel(a, w) for a, w in zip(two, want)]
    record(f"config3 mul d={d} b={b} m=32", UX=e[0], dX=e[1], dV=e[2], UX_two_call=e2[0], dX_two_call=e2[1],
           dV_two_call=e2[2])
    assert max(e + e2) <= TOL, (e, e2)


@pytest.mark.parametrize("d", [3072, 4096])
@pytest.mark.parametrize("op", ["exp", "cayley"])
def test_config3_exp_cayley_large_d_vs_reference(fb, ref, d, op):
    """apply_exponential / apply_cayley (matops.hpp:98,107) on the reference's
    symmetric-form generator (bench.hpp:124-126: sigma ~ U(-0.9, 0.9))."""
    import torch
    if not hasattr(ref, "gen_layer"):
        pytest.skip("needs oracle/_ref for the generator")
    U, V, s, X, _ = ref.gen_layer(0, d, 32, symmetric=True)
    want = ref.matop(1 if op == "exp" else 2, U, V, s, X, 64)
    p = fb.SvdParam(d, d, dev(U), torch.empty(0, d, device="cuda"), dev(s))
    fn = fb.apply_exponential if op == "exp" else fb.apply_cayley
    got = fn(p, dev(X), 64)
    e = rel(got, want)
    record(f"config3 {op} d={d} b=64 m=32", Y=e)
    assert e <= TOL, e


# ---- config [1] as the layer and config [3]: the MLP step at d = 784 ----------

def test_config2_svd_layer_d784_vs_reference(fb, ref):
    """svd_forward + svd_backward (svd_layer.hpp:106-154) at d = 784, b = 32,
    batch 32 on the reference's layer generator (bench.hpp:122-134)."""
    if not hasattr(ref, "gen_layer"):
        pytest.skip("needs oracle/_ref for the generator")
    U, V, s, X, G = ref.gen_layer(0, 784, 32)
    want = ref.svd_fwd_bwd(U, V, s, X, G, 32)
    p = fb.SvdParam(784, 784, dev(U), dev(V), dev(s))
    Y, g = fb.svd_forward_backward(p, dev(X), dev(G), 32)
    got = (Y, g.grad_input, g.grad_U_vectors, g.grad_V_vectors, g.grad_sigma)
    e = [rel(a, w) for a, w in zip(got, want)]
    record("config2 svd layer d=784 b=32 m=32", Y=e[0], dX=e[1], dU=e[2], dV=e[3], dsigma=e[4])
    assert max(e) <= TOL, e


def test_config4_mlp_step_d784_vs_reference(fb, ref):
    """One training step of the depth-4 MLP of d = 784 SVD layers (BASELINE
    configs[3], demos/svd_layer_demo.cpp:25-43 with the log|det| regulariser)
    against the same step composed from the reference's svd_forward /
    svd_backward / svd_step / clamp_sigma (via the oracle)."""
    import torch

    from paper_2009_13977_b200 import mlp
    from tests.test_gpu_mlp import oracle_step

    cfg = mlp.MLPConfig(d=784, depth=4, block_width=32, eta=1e-3, lam=1e-3)
    layers = mlp.random_layers(cfg, seed=11)
    hl = [(p.U.double().cpu().numpy(), p.V.double().cpu().numpy(), p.sigma.double().cpu().numpy())
          for p in layers]
    rng = np.random.default_rng(12)
    x = rng.standard_normal((cfg.d, 32))
    target = rng.standard_normal((cfg.d, 32))
    want, want_loss = oracle_step(hl, x, target, cfg, oracle=ref)
    loss = float(mlp.train_step(layers, torch.tensor(x, dtype=torch.float32, device="cuda"),
                                torch.tensor(target, dtype=torch.float32, device="cuda"), cfg))
    errs = {"loss": abs(loss - want_loss) / abs(want_loss)}
    for k, (p, (U, V, s)) in enumerate(zip(layers, want)):
        errs[f"U{k}"] = rel(p.U, U)
        errs[f"V{k}"] = rel(p.V, V)
        errs[f"sigma{k}"] = rel(p.sigma, s)
    record("config4 mlp step d=784 depth=4 b=32 m=32", **errs)
    assert max(errs.values()) <= TOL, errs


# ---- config [4] and the large-batch route -------------------------------------

def _uses_large_batch(d, n, m):
    """capi.cpp's path selection (exported for diagnostics)."""
    import ctypes as C

    from paper_2009_13977_b200 import _lib
    f = _lib.load().use_large_batch
    f.restype, f.argtypes = C.c_bool, [C.c_int] * 3
    return bool(f(d, n, m))


def _large_batch_vs_reference(fb, ref, d, m, b, label, seed):
    """UX, dX and dV over the whole batch against the reference (one oracle
    call: its cost is the 8192-column CPU FastH, ~1 min on 16 host threads)."""
    import torch
    rng = np.random.default_rng(seed)
    V = rng.standard_normal((d, d))
    X = rng.standard_normal((d, m))
    G = rng.standard_normal((d, m))
    Y, back = fb.fasth_forward_backward(dev(V), dev(X), dev(G), b)
    torch.cuda.synchronize()
    want = ref.fasth_fwd_bwd(V, X, G, b)
    e = [rel(a, w) for a, w in zip((Y, back.grad_input, back.grad_vectors), want)]
    record(label, UX=e[0], dX=e[1], dV=e[2])
    return e


def test_config5_shape_vs_reference(fb, ref):
    """BASELINE configs[4]'s per-GPU shape: d = 2048, batch 8192 (the tcgen05
    large-batch path, chosen by default)."""
    assert fb is not None
    assert _uses_large_batch(2048, 2048, 8192)
    e = _large_batch_vs_reference(fb, ref, 2048, 8192, 32, "config5 d=2048 m=8192 b=32", 5)
    assert max(e) <= TOL, e


@pytest.mark.parametrize("m", [64, 1024])
def test_large_batch_default_route_d4096(fb, ref, m):
    """The default large-batch route at d = 4096 (capi.cpp use_large_batch:
    m >= 64 at d >= 4096), the longest accumulation chains (K = d) of the
    tcgen05 products."""
    assert _uses_large_batch(4096, 4096, m)
    e = _large_batch_vs_reference(fb, ref, 4096, m, 64, f"large-batch route d=4096 m={m} b=64", 40 + m)
    assert max(e) <= TOL, e


# ---- shapes the reference accepts (fasth.hpp:40-61: any d, n, m, b) -----------

@pytest.mark.parametrize("d,n,m,b", [(5000, 5000, 32, 64), (8192, 8192, 32, 64), (2048, 2000, 1000, 32),
                                     (1024, 8320, 128, 32)])
def test_any_shape_vs_reference(fb, ref, d, n, m, b):
    """Shapes past the chain kernels' reach (d > 4096) or off the tcgen05
    path's alignment (n not a multiple of 128, more than 64 WY stages): the
    large-batch path on zero-padded dimensions (lb.h Dims)."""
    rng = np.random.default_rng(d + n + m)
    V = rng.standard_normal((n, d))
    X = rng.standard_normal((d, m))
    G = rng.standard_normal((d, m))
    Y, back = fb.fasth_forward_backward(dev(V), dev(X), dev(G), b)
    tape = fb.fasth_forward(dev(V), dev(X), b)
    two = fb.fasth_backward(tape, dev(G))
    want = ref.fasth_fwd_bwd(V, X, G, b)
    e = [rel(a, w) for a, w in zip((Y, back.grad_input, back.grad_vectors), want)]
    e2 = [rel(a, w) for a, w in zip((tape.output(), two.grad_input, two.grad_vectors), want)]
    record(f"shape d={d} n={n} m={m} b={b}", UX=e[0], dX=e[1], dV=e[2], UX_two_call=e2[0], dX_two_call=e2[1],
           dV_two_call=e2[2])
    assert max(e + e2) <= TOL, (e, e2)


@pytest.mark.parametrize("d,n,m", [(1001, 999, 130), (300, 200, 5), (130, 129, 17), (64, 64, 32)])
def test_ragged_shapes_forced_large_batch(fb, ref, d, n, m, monkeypatch):
    """Ragged d (not a multiple of 4), n and m on the tcgen05 path (forced with
    FASTH_LB=1) against the reference, one-call and two-call."""
    monkeypatch.setenv("FASTH_LB", "1")
    rng = np.random.default_rng(3 * d + n + m)
    V = rng.standard_normal((n, d))
    X = rng.standard_normal((d, m))
    G = rng.standard_normal((d, m))
    Y, back = fb.fasth_forward_backward(dev(V), dev(X), dev(G), 16)
    tape = fb.fasth_forward(dev(V), dev(X), 16)
    two = fb.fasth_backward(tape, dev(G))
    want = ref.fasth_fwd_bwd(V, X, G, 16)
    e = [rel(a, w) for a, w in zip((Y, back.grad_input, back.grad_vectors), want)]
    e2 = [rel(a, w) for a, w in zip((tape.output(), two.grad_input, two.grad_vectors), want)]
    record(f"forced large-batch d={d} n={n} m={m}", UX=e[0], dX=e[1], dV=e[2])
    assert max(e + e2) <= TOL, (e, e2)


# ---- apply_pseudo_inverse (matops.hpp:158), rectangular ---------------------------

@pytest.mark.parametrize("out_dim,in_dim,m,tol", [(784, 784, 32, 0.0), (96, 64, 8, 0.6), (64, 96, 5, 0.6),
                                                  (300, 300, 17, 1.0)])
def test_apply_pseudo_inverse_vs_reference(fb, ref, out_dim, in_dim, m, tol):
    if not hasattr(ref, "pinv"):
        pytest.skip("needs oracle/_ref")
    U, V, s, _, _ = ref.gen_param(7 + out_dim, out_dim, in_dim, out_dim, in_dim, m)
    X = np.random.default_rng(out_dim + in_dim).standard_normal((out_dim, m))
    want = ref.pinv(U, V, s, X, tol, 32, out_dim, in_dim)
    p = fb.SvdParam(out_dim, in_dim, dev(U), dev(V), dev(s))
    got = fb.apply_pseudo_inverse(p, dev(X), tol, 32)
    e = rel(got, want)
    record(f"apply_pseudo_inverse {out_dim}x{in_dim} m={m} tol={tol}", Y=e)
    assert e <= TOL, e
    with pytest.raises(fb.Error):
        fb.apply_pseudo_inverse(p, dev(X), -1.0, 32)
