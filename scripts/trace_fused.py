"""One traced pipelined fasth_forward_backward at (d, b, m) under FASTH_TRACE
(build phase stamps + global timers, sweep step stamps), for
scripts/trace_report.py --timeline."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_2009_13977_b200 import fasth as fb

d, b, m = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (784, 32, 32)))
V = torch.randn(d, d, device="cuda")
X = torch.randn(m, d, device="cuda").t()
G = torch.randn(m, d, device="cuda").t()
for _ in range(3):
    fb.fasth_forward_backward(V, X, G, b)
torch.cuda.synchronize()
