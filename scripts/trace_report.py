"""Summarise FASTH_TRACE sweep dumps: cycles per phase per step (chain_sweep.cu
slots: 0 top, 1 A after load wait, 2 A done, 3 B after exchange wait,
4 B done, 5 after barrier 1, 6 C done, 7 after barrier 2).  Slots 0-2,5-7
are stamped by thread 0 (an A warp), 3-4 by the first B warp: all on the same
SM clock."""
import sys
import numpy as np


def report(path):
    raw = open(path, "rb").read()
    nctas, q = np.frombuffer(raw[:8], dtype=np.int32)
    tr = np.frombuffer(raw[8:], dtype=np.int64).reshape(nctas, q + 1, 16).astype(np.float64)
    s = tr[:, :q, :]
    print(f"{path}: {nctas} CTAs, q={q}")
    print(f"  cycles/step (top to top): {np.mean(np.diff(s[:, :, 0], axis=1)):.0f}")
    rows = [("A load wait", 1, 0, slice(0, q - 1)), ("A partial+push", 2, 1, slice(0, q - 1)),
            ("B exch wait (from top)", 3, 0, slice(1, q)), ("B reduce+corr", 4, 3, slice(1, q)),
            ("barrier1 (from A done)", 5, 2, slice(0, q - 1)), ("barrier1 (from B done)", 5, 4, slice(1, q)),
            ("C update", 6, 5, slice(0, q)), ("barrier2+refill", 7, 6, slice(0, q)),
            ("  A: mma loop", 8, 1, slice(0, q - 1)), ("  A: chunk combine", 9, 8, slice(0, q - 1)),
            ("  A: push", 2, 9, slice(0, q - 1))]
    for name, k1, k0, sl in rows:
        v = s[:, sl, k1] - s[:, sl, k0]
        print(f"  {name:26s} mean {v.mean():7.0f}  p50 {np.median(v):7.0f}  max {v.max():7.0f}")


for p in sys.argv[1:]:
    report(p)
