"""Summarise FASTH_TRACE sweep dumps: cycles per phase per step.

v1 (chain_kernel.cu, *.fwd.bin / *.bwd.bin) slots: 0 top, 1 A after load
wait, 2 A done, 3 B after exchange wait, 4 B done, 5 after barrier 1, 6 C
done, 7 after barrier 2, 8 A mma loop done, 9 A chunk combine done.
v2 (chain_v2.cu, *.v2.bin) slots: 0 top, 1 partial MMAs done (before the
combine barrier), 2 row warps' phase 1 done (pushed), 3 B after exchange
wait, 4 B done, 5 after barrier 1, 6 update done, 7 after barrier 2.
Slots 0-2, 5-7 are stamped by thread 0 (row warp 0), 3-4 by the first B
warp: the same SM clock.  Note BAR.SYNC defers its block to the next
dependent instruction, so a stamp right after a barrier is its issue time."""
import sys

import numpy as np


def report_build(path):
    raw = open(path, "rb").read()
    n, k = np.frombuffer(raw[:8], dtype=np.int32)
    tr = np.frombuffer(raw[8:], dtype=np.int64).reshape(n, k).astype(np.float64)
    tr = tr[tr[:, 0] != 0]  # blocks this launch did not build (persistent builders) stay zero
    n = len(tr)
    names = ["load V rows", "Gram band", "cluster reduce", "degeneracy+mask", "T~ + B operands", "W rows", "stores"]
    print(f"{path}: {n} CTAs; build phases (cycles, mean / max over CTAs); total mean {np.mean(tr[:, 7] - tr[:, 0]):.0f}")
    for j, nm in enumerate(names):
        v = tr[:, j + 1] - tr[:, j]
        print(f"  {nm:22s} mean {v.mean():7.0f}  max {v.max():7.0f}")
    t0 = tr[:, 0].min()
    print(f"  CTA start spread: {tr[:, 0].max() - t0:.0f} cycles (same-SM clocks only comparable)")


def report_warps(path, nr=None):
    """Per-warp barrier arrivals of the v2 sweep: which role arrives last at
    each CTA barrier (the step's critical path) and how long each barrier
    takes to release after its last arrival."""
    raw = open(path, "rb").read()
    nctas, q = np.frombuffer(raw[:8], dtype=np.int32)
    w = np.frombuffer(raw[8:], dtype=np.int64).reshape(nctas, q, 12, 4).astype(np.float64)
    used = np.where(w[:, :, :, 0].max(axis=(0, 1)) != 0)[0]
    w = w[:, 1:q - 1, used, :]  # interior steps
    nw = len(used)
    print(f"{path}: {nctas} CTAs, {nw} warps (row warps, B warps, producer)")
    for bi, (ka, kr) in enumerate(((0, 1), (2, 3))):
        arr = w[:, :, :, ka]
        last = arr.max(axis=2)
        rel = w[:, :, :, kr].min(axis=2)
        lag = last[:, :, None] - arr  # how long before the last arrival each warp arrived
        print(f"  barrier {bi + 1}: release - last arrival mean {np.mean(rel - last):.0f} cycles; "
              f"mean slack per warp (cycles before the last arrival): " +
              " ".join(f"w{u}:{lag[:, :, j].mean():.0f}" for j, u in enumerate(used)))
    # step = release S2 (t) -> release S2 (t+1)
    r2 = w[:, :, :, 3].min(axis=2)
    print(f"  step (S2 release to S2 release): {np.mean(np.diff(r2, axis=1)):.0f} cycles; "
          f"S2 release -> last arrival at S1: {np.mean(w[:, 1:, :, 0].max(axis=2) - r2[:, :-1]):.0f}; "
          f"S1 release -> last arrival at S2: {np.mean(w[:, :, :, 2].max(axis=2) - w[:, :, :, 1].min(axis=2)):.0f}")


def report(path):
    if path.endswith(".warps.bin"):
        return report_warps(path)
    if path.endswith(".build.bin"):
        return report_build(path)
    raw = open(path, "rb").read()
    nctas, q = np.frombuffer(raw[:8], dtype=np.int32)
    tr = np.frombuffer(raw[8:], dtype=np.int64).reshape(nctas, q + 1, 16).astype(np.float64)
    s = tr[:, :q, :]
    print(f"{path}: {nctas} CTAs, q={q}")
    print(f"  cycles/step (top to top): {np.mean(np.diff(s[:, :, 0], axis=1)):.0f}"
          f"   whole sweep (top 0 -> after last barrier): {np.mean(s[:, q - 1, 7] - s[:, 0, 0]):.0f}")
    if path.endswith(".v2.bin"):
        g = tr[:, q, :]
        t0 = g[:, 10]
        names = {11: "X loaded", 12: "cluster synced", 13: "prologue pushed", 14: "loop done", 15: "exit"}
        print("  prologue/epilogue (ns from kernel entry, mean over CTAs): " +
              ", ".join(f"{v} {np.mean(g[:, k] - t0):.0f}" for k, v in names.items()))
        print(f"  loop: step 0 top at {np.mean(s[:, 0, 8] - t0):.0f} ns, last step end at {np.mean(s[:, q - 1, 9] - t0):.0f} ns")
        rows = [("row: partial MMAs", 1, 0, slice(0, q - 1)), ("row: combine+push", 2, 1, slice(0, q - 1)),
                ("B: exch wait (from top)", 3, 0, slice(0, q)), ("B: reduce+scatter", 4, 3, slice(0, q)),
                ("barrier1 (from row done)", 5, 2, slice(0, q)), ("barrier1 (from B done)", 5, 4, slice(0, q)),
                ("update", 6, 5, slice(0, q)), ("barrier2", 7, 6, slice(0, q))]
        if (s[:, :, 10] != 0).any():  # B-warp detail stamps (chain_v2.cu slots 10, 11)
            rows[4:4] = [("  B: re-arm + S.Z result", 10, 3, slice(0, q)), ("  B: sum of C partials", 11, 10, slice(0, q)),
                         ("  B: scatter (+ Z' stores)", 4, 11, slice(0, q))]
    else:
        rows = [("A load wait", 1, 0, slice(0, q - 1)), ("A partial+push", 2, 1, slice(0, q - 1)),
                ("B exch wait (from top)", 3, 0, slice(1, q)), ("B reduce+corr", 4, 3, slice(1, q)),
                ("barrier1 (from A done)", 5, 2, slice(0, q - 1)), ("barrier1 (from B done)", 5, 4, slice(1, q)),
                ("C update", 6, 5, slice(0, q)), ("barrier2+refill", 7, 6, slice(0, q)),
                ("  A: mma loop", 8, 1, slice(0, q - 1)), ("  A: chunk combine", 9, 8, slice(0, q - 1)),
                ("  A: push", 2, 9, slice(0, q - 1))]
    for name, k1, k0, sl in rows:
        v = s[:, sl, k1] - s[:, sl, k0]
        if v.size:
            print(f"  {name:26s} mean {v.mean():7.0f}  p50 {np.median(v):7.0f}  max {v.max():7.0f}")


def timeline(build_path, sweep_path):
    """Global-timer view of a pipelined step: when each WY block became ready
    (last of its CTAs) vs when the sweeps started each step (ns)."""
    raw = open(build_path, "rb").read()
    n, k = np.frombuffer(raw[:8], dtype=np.int32)
    b = np.frombuffer(raw[8:], dtype=np.int64).reshape(n, k)
    raw = open(sweep_path, "rb").read()
    nc, q = np.frombuffer(raw[:8], dtype=np.int32)
    s = np.frombuffer(raw[8:], dtype=np.int64).reshape(nc, q + 1, 16)
    C = n // q
    t0 = min(b[:, 8][b[:, 8] > 0].min(), s[:, 0, 8].min())
    ready = (b[:, 9].reshape(q, C).max(axis=1) - t0) / 1e3
    start = (b[:, 8].reshape(q, C).min(axis=1) - t0) / 1e3
    print(f"timeline (us from first build CTA start), q={q}")
    print("  block build start : " + " ".join(f"{x:5.1f}" for x in start))
    print("  block ready       : " + " ".join(f"{x:5.1f}" for x in ready))
    half = nc // 2
    for name, rows in (("fwd", slice(0, half)), ("bwd", slice(half, nc))):
        st = (s[rows, :q, 8].min(axis=0) - t0) / 1e3
        en = (s[rows, :q, 9].max(axis=0) - t0) / 1e3
        print(f"  {name} step start    : " + " ".join(f"{x:5.1f}" for x in st))
        print(f"  {name} step end      : " + " ".join(f"{x:5.1f}" for x in en))


if __name__ == "__main__":
    if sys.argv[1] == "--timeline":
        timeline(sys.argv[2], sys.argv[3])
    else:
        for p in sys.argv[1:]:
            report(p)
