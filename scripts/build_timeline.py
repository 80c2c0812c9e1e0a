"""Global-timer view of one traced build launch (FASTH_TRACE *.build.bin):
per block, when its first CTA started and its last CTA ended (us from the
first CTA start) -- shows waves and per-block latency."""
import sys

import numpy as np

raw = open(sys.argv[1], "rb").read()
n, k = np.frombuffer(raw[:8], dtype=np.int32)
tr = np.frombuffer(raw[8:], dtype=np.int64).reshape(n, k).astype(np.float64)
q = int(sys.argv[2]) if len(sys.argv) > 2 else 25
C = n // q
g0 = tr[:, 8].reshape(q, C)
g1 = tr[:, 9].reshape(q, C)
t0 = g0.min()
st, en = (g0.min(axis=1) - t0) / 1e3, (g1.max(axis=1) - t0) / 1e3
print(f"{n} CTAs, {q} blocks x {C}; build span {(g1.max() - t0) / 1e3:.2f} us")
print("  block start us: " + " ".join(f"{x:5.2f}" for x in st))
print("  block end   us: " + " ".join(f"{x:5.2f}" for x in en))
print("  CTA start spread within a block (us): mean %.2f max %.2f" % (((g0.max(1) - g0.min(1)) / 1e3).mean(), ((g0.max(1) - g0.min(1)) / 1e3).max()))
ph = np.diff(tr[:, :8], axis=1)
names = ["load", "gram", "reduce", "degen", "T+B", "Wrows", "stores"]
print("  phase cycles mean: " + " ".join(f"{nm}={ph[:, j].mean():.0f}" for j, nm in enumerate(names)))
print("  phase cycles max : " + " ".join(f"{nm}={ph[:, j].max():.0f}" for j, nm in enumerate(names)))
