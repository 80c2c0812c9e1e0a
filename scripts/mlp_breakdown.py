"""Per-kernel breakdown of the config-4 MLP training step (ctx timing mode)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_2009_13977_b200 import fasth as fb
from paper_2009_13977_b200.mlp import MLPConfig, random_layers, train_step

cfg = MLPConfig()
layers = random_layers(cfg)
ctx = fb.Context(0, deferred=True)
x = torch.randn(32, cfg.d, device="cuda").t()
t = torch.randn(32, cfg.d, device="cuda").t()
for _ in range(3):
    train_step(layers, x, t, cfg, ctx=ctx)
torch.cuda.synchronize()
R = 10
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(R):
    train_step(layers, x, t, cfg, ctx=ctx)
e1.record()
torch.cuda.synchronize()
print(f"step {e0.elapsed_time(e1) * 1e3 / R:.1f} us (eager)")
ctx.set_timing(True)
for _ in range(R):
    train_step(layers, x, t, cfg, ctx=ctx)
torch.cuda.synchronize()
kt = ctx.kernel_times()
ctx.set_timing(False)
for k, (ms, n) in sorted(kt.items(), key=lambda x: -x[1][0]):
    print(f"{k:24s} {ms * 1e3 / R:8.1f} us/step ({n // R} launches)")
