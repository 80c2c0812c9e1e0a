"""Timeline of one fused step (FASTH_STEPTRACE dump, <path>.bin): per-kernel
global-timer windows of the builder, the sweep and the gradient kernel, us
from the first builder CTA's start.  usage: step_timeline.py <path>.bin"""
import sys

import numpy as np

raw = open(sys.argv[1], "rb").read()
q, C, brows, sctas, dctas, valid = np.frombuffer(raw[:24], dtype=np.int32)
a = np.frombuffer(raw[24:], dtype=np.int64).astype(np.float64)
b = a[:brows * 10].reshape(brows, 10)
o = brows * 10
s = a[o:o + sctas * (q + 1) * 16].reshape(sctas, q + 1, 16)
o += sctas * (q + 1) * 16
dv = a[o:o + dctas * 6].reshape(dctas, 6)
t0 = b[:, 8].min()
us = lambda x: (x - t0) / 1e3  # noqa: E731
print(f"q={q} C={C}: {brows} builder CTAs, {sctas} sweep CTAs, {dctas} gradient CTAs (us from first builder start)")
print(f"  builder : start {us(b[:, 8].min()):6.2f}..{us(b[:, 8].max()):6.2f}  end {us(b[:, 9].min()):6.2f}..{us(b[:, 9].max()):6.2f}")
if brows % q == 0:
    be = b[:, 9].reshape(q, brows // q).max(axis=1)
    print("  builder end per block: " + " ".join(f"{x:5.1f}" for x in us(be)))
r = s[:, q, :]
for k, nm in ((10, "entry"), (11, "X loaded"), (12, "cluster synced"), (13, "prologue pushed"), (14, "loop done"), (15, "exit")):
    v = r[:, k]
    v = v[v > 0]
    if v.size:
        print(f"  sweep {nm:16s}: {us(v.min()):6.2f}..{us(v.max()):6.2f}")
st = s[:, :q, 8]
en = s[:, :q, 9]
if (st > 0).all():
    print("  sweep step start (min over CTAs): " + " ".join(f"{x:5.1f}" for x in us(st.min(axis=0))))
    per = np.diff(st.min(axis=0))
    print(f"  sweep mean step {per.mean() * 1e-3:.3f} us")
if dctas:
    d = dv[dv[:, 0] > 0]
    print(f"  dv entry   {us(d[:, 0].min()):6.2f}..{us(d[:, 0].max()):6.2f}")
    print(f"  dv go      {us(d[:, 1].min()):6.2f}..{us(d[:, 1].max()):6.2f}")
    print(f"  dv loaded  {us(d[:, 2].min()):6.2f}..{us(d[:, 2].max()):6.2f}  (go->loaded mean {np.mean(d[:, 2] - d[:, 1]) / 1e3:.2f} us)")
    print(f"  dv V-term  {us(d[:, 3].min()):6.2f}..{us(d[:, 3].max()):6.2f}  (loaded->V mean {np.mean(d[:, 3] - d[:, 2]) / 1e3:.2f} us)")
    print(f"  dv end     {us(d[:, 4].min()):6.2f}..{us(d[:, 4].max()):6.2f}  (V->end mean {np.mean(d[:, 4] - d[:, 3]) / 1e3:.2f} us)")
    print(f"  dv SMs used {len(set(d[:, 5].astype(int)))}")
    if dctas % q == 0 and (dv[:, 4] > 0).all():
        de = dv[:, 4].reshape(q, dctas // q).max(axis=1)
        print("  dv end per block: " + " ".join(f"{x:5.1f}" for x in us(de)))
