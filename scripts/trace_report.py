"""Summarise FASTH_TRACE sweep dumps: mean cycles per phase per step.
phases (chain_sweep.cu marks): 0 top, 1 after load wait, 2 after partial+push,
3 after exchange wait, 4 after reduce (B), 5 after update (C), 6 end of step."""
import sys
import numpy as np


def report(path):
    raw = open(path, "rb").read()
    nctas, q = np.frombuffer(raw[:8], dtype=np.int32)
    tr = np.frombuffer(raw[8:], dtype=np.int64).reshape(nctas, q + 1, 8)
    names = ["tape/top->loadwait", "partial+push", "exch wait", "reduce B", "update C", "tape+refill"]
    print(f"{path}: {nctas} CTAs, q={q}")
    tot = tr[:, q - 1, 6] - tr[:, q, 1]
    print(f"  prologue (L0) cycles: mean {np.mean(tr[:, q, 1] - tr[:, q, 0]):.0f}; steps total mean {np.mean(tot):.0f} "
          f"-> {np.mean(tot) / q:.0f} cycles/step")
    steps = tr[:, :q, :]
    d = {}
    d[names[0]] = steps[:, :-1, 1] - steps[:, :-1, 0]
    d[names[1]] = steps[:, :-1, 2] - steps[:, :-1, 1]
    d[names[2]] = steps[:, :, 3] - steps[:, :, 2]
    d[names[3]] = steps[:, :, 4] - steps[:, :, 3]
    d[names[4]] = steps[:, :, 5] - steps[:, :, 4]
    d[names[5]] = steps[:, :, 6] - steps[:, :, 5]
    for k, v in d.items():
        print(f"  {k:22s} mean {v.mean():8.0f}  p50 {np.median(v):8.0f}  max {v.max():8.0f}")


for p in sys.argv[1:]:
    report(p)
