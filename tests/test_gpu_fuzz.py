"""Seeded random shapes through the default path selection (cluster chain
sweep, panel sweep or the large-batch tcgen05 path, whichever capi.cpp picks)
against the float64 blocked model of tests/test_gpu_lb.py.  The shapes are
drawn to hit the corners the fixed cases do not: vector counts above and
below d, d not a multiple of 4, batch 1, block sizes that do not divide n,
and sizes on either side of the large-batch thresholds."""
import numpy as np
import pytest
import torch

from tests.test_gpu_lb import TOL, model64, rel

pytestmark = pytest.mark.gpu


def _shapes(count=24, seed=2009):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(count):
        d = int(rng.choice([int(rng.integers(1, 130)), int(rng.integers(130, 1100)), int(rng.integers(1000, 2100))]))
        if i % 3 == 0:
            d = max(128, d // 4 * 4)  # large-batch eligible geometry
        n = int(rng.choice([d, int(rng.integers(1, d + 1)), int(rng.integers(d, 2 * d + 1))]))
        m = int(rng.choice([1, int(rng.integers(1, 65)), int(rng.integers(64, 600)), int(rng.integers(1000, 3000))]))
        if i % 3 == 0:
            m = max(16, m // 4 * 4)
            n = max(128, n // 128 * 128)
        b = int(rng.choice([32, int(rng.integers(1, 129))]))
        out.append((n, d, m, b))
    return out


@pytest.mark.parametrize("n,d,m,b", _shapes())
def test_random_shape_matches_f64(n, d, m, b):
    from paper_2009_13977_b200 import fasth as fb
    g = torch.Generator(device="cuda").manual_seed(n * 7919 + d * 31 + m)
    V = torch.randn(n, d, device="cuda", generator=g)
    X = torch.randn(m, d, device="cuda", generator=g).t()
    G = torch.randn(m, d, device="cuda", generator=g).t()
    Y, back = fb.fasth_forward_backward(V, X, G, b)
    torch.cuda.synchronize()
    Yr, dXr, dVr = model64(V, X, G, 64)
    errs = (rel(Y, Yr), rel(back.grad_input, dXr), rel(back.grad_vectors, dVr))
    print(f"n={n} d={d} m={m} b={b}: rel err Y {errs[0]:.2e} dX {errs[1]:.2e} dV {errs[2]:.2e}")
    assert all(np.isfinite(errs)) and max(errs) <= TOL, errs
