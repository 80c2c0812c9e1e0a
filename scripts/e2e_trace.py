"""Timeline of the host-buffer step (FASTH_STEPTRACE must be set): runs
fasth_forward_backward_host a few times, dumps the last call's builder /
sweep / gradient windows."""
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2009_13977_b200 import fasth as fb  # noqa: E402

d, m, b = 784, 32, 32
torch.manual_seed(0)
Vh, Xh, Gh = torch.randn(d, d).pin_memory(), torch.randn(m, d).pin_memory(), torch.randn(m, d).pin_memory()
ctx = fb.Context(0)
out = tuple(torch.empty(s).pin_memory() for s in ((m, d), (m, d), (d, d)))
for _ in range(10):
    t0 = time.perf_counter()
    fb.forward_backward_host(Vh, Xh, Gh, b, ctx=ctx, out=out)
    t1 = time.perf_counter()
print(f"last call wall {1e6 * (t1 - t0):.1f} us")
ctx.check()
print(subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "step_timeline.py"),
                      os.environ["FASTH_STEPTRACE"] + ".bin"], capture_output=True, text=True).stdout)
