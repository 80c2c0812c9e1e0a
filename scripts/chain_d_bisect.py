"""Probe: chain-kernel path vs the tcgen05 path (FASTH_LB=1) over d at batch
32, under the chain path's variant knobs, to localise a d-dependent defect."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_13977_b200 import fasth as fb  # noqa: E402


def run(V, X, G, b, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        Y, back = fb.fasth_forward_backward(V, X, G, b)
        torch.cuda.synchronize()
        return Y.clone(), back.grad_input.clone(), back.grad_vectors.clone()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def rel(a, b):
    return float((a.double() - b.double()).norm() / max(b.double().norm(), 1.0))


ds = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [3200, 3584, 3840, 3968, 4032, 4064, 4096]
# (round 2 localised the d > 3072 defect with the first-generation builder /
# sweep / gradient kernels as alternates; those kernels are gone since)
variants = {"chain": {}, "no_pdl": {"FASTH_NO_PDL": "1"}}
for d in ds:
    g = torch.Generator(device="cuda").manual_seed(d)
    V = torch.randn(d, d, device="cuda", generator=g)
    X = torch.randn(32, d, device="cuda", generator=g).t()
    G = torch.randn(32, d, device="cuda", generator=g).t()
    want = run(V, X, G, 32, {"FASTH_LB": "1"})
    for name, env in variants.items():
        env = dict(env, FASTH_LB="0")
        try:
            got = run(V, X, G, 32, env)
            print(d, name, ["%.2e" % rel(a, w) for a, w in zip(got, want)], flush=True)
        except Exception as e:  # noqa: BLE001
            print(d, name, "error", str(e)[:120], flush=True)
