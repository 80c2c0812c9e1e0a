"""One traced fwd+bwd at (d, b, m) under FASTH_TRACE, for scripts/trace_report.py."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

from paper_2009_13977_b200 import fasth as fb

d, b, m = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (784, 32, 32)))
rng = np.random.default_rng(0)
V = torch.tensor(rng.standard_normal((d, d)), dtype=torch.float32, device="cuda")
X = torch.tensor(rng.standard_normal((d, m)), dtype=torch.float32, device="cuda")
G = torch.tensor(rng.standard_normal((d, m)), dtype=torch.float32, device="cuda")
for _ in range(3):  # warm
    t = fb.fasth_forward(V, X, b)
    fb.fasth_backward(t, G)
torch.cuda.synchronize()
