"""fasth-bench for the B200 path: the reference CLI (tools/fasth_bench.cpp:23-42,
81-90) with the same flags and CSV records (bench.hpp:67), timing the GPU
implementation.

    python tools/fasth_bench_b200.py --d 64,128,256 --algo fasth --reps 100
    python tools/fasth_bench_b200.py --d 256:256:4 --op inverse --k auto --out r.csv
    python tools/fasth_bench_b200.py --verify

Algorithms: ``fasth`` (this library on cuda:0), ``ref-fasth`` / ``ref-sequential``
(the unmodified reference's CPU run_bench, oracle/_ref, for baselines in the
same file).  Ops: mul | layer | det | inverse | exp | cayley, with the
reference's workloads (bench.hpp:117-209: mt19937_64(seed + d), the derived
SVD-form parameter for the matrix operations).  The checksum column of the
reference (bench.hpp:94-108, exact f64 only) is replaced by ``rel_err``: the
Frobenius-relative error of the forward output against the reference's f64
result (matrix.hpp:106-110); added columns: gpus, tflops, roofline_frac
(F_alg = 12 d n m + 4 d n b per fwd+bwd, 2x for a layer, against the 3xTF32
peak derived from MEASURED_PEAKS.json).

Exit codes as the reference: 0 success, 1 configuration error, 2 verification
failure.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

HEADER = "algo,op,d,m,k,reps,threads,mean_s,std_s,rel_err,gpus,tflops,roofline_frac"
OPS = ("mul", "inverse", "det", "exp", "cayley", "layer")


def parse_dims(spec: str) -> list[int]:
    """tools/fasth_bench.cpp:23-42: comma list or start:step:count."""
    if ":" in spec:
        parts = spec.split(":")
        if len(parts) != 3 or not all(p.strip().isdigit() for p in parts):
            raise ValueError(f"--d: expected start:step:count, got '{spec}'")
        start, step, count = (int(p) for p in parts)
        return [start + i * step for i in range(count)]
    return [int(t) for t in spec.split(",") if t]


def peak_3xtf32() -> float:
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"] / 6.0
    except Exception:
        return 1590.0 / 6.0


def workload(op: str, d: int, m: int, seed: int):
    """The reference's synthetic data for (op, d) (bench.hpp:117-135)."""
    from oracle.oracle import Ref
    R = Ref()
    if op == "mul":
        V, X, G = R.gen_mul(seed, d, m)
        return {"V": V, "X": X, "G": G}
    U, V, s, X, G = R.gen_layer(seed, d, m, symmetric=op in ("exp", "cayley"))
    return {"U": U, "V": V, "sigma": s, "X": X, "G": G}


def derive(op: str, w):
    """bench.hpp:160-185: the SVD-form parameter each matrix operation times."""
    import numpy as np
    U, V, s = w["U"], w["V"], w["sigma"]
    if op in ("layer", "det"):
        return U, V, s
    if op == "inverse":
        return V, U, 1.0 / s
    f = np.exp(s) if op == "exp" else (1.0 - s) / (1.0 + s)
    return U, U, f


def reference_output(op: str, w, b: int):
    from oracle.oracle import Ref
    R = Ref()
    if op == "mul":
        return R.fasth_fwd_bwd(w["V"], w["X"], w["G"], b)[0]
    U, V, s = derive(op, w)
    d = w["X"].shape[0]
    return R.svd_fwd_bwd(U, V, s, w["X"], w["G"], b, out_dim=d, in_dim=d)[0]


def time_fasth(op: str, w, b: int, reps: int):
    """Device seconds per repetition (CUDA events, mean and std over reps)."""
    import numpy as np
    import torch

    from paper_2009_13977_b200 import fasth as fb
    dev = torch.device("cuda", 0)
    t = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float32, device=dev)
    X, G = t(w["X"]), t(w["G"])
    ctx = fb.Context(0, deferred=True)
    if op == "mul":
        V = t(w["V"])

        def step():
            return fb.fasth_forward_backward(V, X, G, b, ctx=ctx)[0]
    else:
        U, Vv, s = derive(op, w)
        d = w["X"].shape[0]
        p = fb.SvdParam(d, d, t(U), t(Vv) if Vv.size else torch.empty(0, d, device=dev), t(s))

        def step():
            if op == "det":  # bench.hpp:162: log|det| of the parameter, then the layer
                fb.log_abs_det(p, ctx=ctx)
            # G drawn up front (bench.hpp:166-209): the paired-sweep layer call
            y, _ = fb.svd_forward_backward(p, X, G, b, ctx=ctx)
            return y
    y = step()
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        e.record()
        e.synchronize()
        times.append(a.elapsed_time(e) * 1e-3)
    ctx.check()
    mean = sum(times) / len(times)
    std = math.sqrt(sum((x - mean) ** 2 for x in times) / max(len(times) - 1, 1))
    return mean, std, y.double().cpu().numpy()


def run(args) -> int:
    import numpy as np

    from oracle.oracle import Ref, relative_error
    dims = parse_dims(args.d)
    algos = [a for a in args.algo.split(",") if a]
    for a in algos:
        if a not in ("fasth", "ref-fasth", "ref-sequential"):
            print(f"--algo: unknown algorithm '{a}'", file=sys.stderr)
            return 1
    if args.op not in OPS:
        print(f"--op: expected one of {'|'.join(OPS)}", file=sys.stderr)
        return 1
    out = open(args.out, "w") if args.out else sys.stdout
    print(HEADER, file=out)
    peak = peak_3xtf32()
    for d in dims:
        w = workload(args.op, d, args.m, args.seed)
        if args.k == "auto":
            if "fasth" in algos:
                from paper_2009_13977_b200 import fasth as fb
                b = fb.tune_block_width(d, args.m, timed=True, seed=args.seed)
            else:
                b = max(1, round(math.sqrt(d)))
        else:
            b = int(args.k)
        ref_y = reference_output(args.op, w, b) if args.check else None
        flops = (12.0 * d * d * args.m + 4.0 * d * d * b) * (1 if args.op == "mul" else 2)
        for algo in algos:
            if algo == "fasth":
                mean, std, y = time_fasth(args.op, w, b, args.reps)
                err = relative_error(y, ref_y) if ref_y is not None else float("nan")
                gpus, threads = 1, 0
            else:
                R = Ref()
                mean, std, _ = R.run_bench(args.op, algo.split("-", 1)[1], d, args.m, b, args.reps, args.seed,
                                           args.threads)
                err, gpus, threads = 0.0, 0, args.threads or R.hardware_threads()
            tf = flops / mean / 1e12
            print(f"{algo},{args.op},{d},{args.m},{b},{args.reps},{threads},{mean:.9g},{std:.9g},"
                  f"{err:.3e},{gpus},{tf:.4f},{tf / peak if gpus else 0.0:.5f}", file=out, flush=True)
    if out is not sys.stdout:
        out.close()
    return 0


def run_verify() -> int:
    """The reference's verification suite (bench.hpp:335-385) restated against
    the GPU path: forward and backward equivalence with the reference's f64
    sequential product on its seeded workloads, plus the SVD layer."""
    import numpy as np
    import torch

    from oracle.oracle import Ref, relative_error
    from paper_2009_13977_b200 import fasth as fb
    R = Ref()
    checks = []
    t = lambda a: torch.tensor(np.ascontiguousarray(a), dtype=torch.float32, device="cuda")
    for d, b in ((16, 4), (64, 8), (64, 64), (100, 7), (256, 32)):
        V, X, G = R.gen_mul(0, d, 8)
        want = R.sequential_fwd_bwd(V, X, G)
        y, back = fb.fasth_forward_backward(t(V), t(X), t(G), b)
        got = (y, back.grad_input, back.grad_vectors)
        for name, g_, w_ in zip(("forward", "backward dX", "backward dV"), got, want):
            e = relative_error(g_.double().cpu().numpy(), w_)
            checks.append((f"{name} d={d} b={b}", e <= 1e-4, f"rel {e:.2e}"))
    U, Vv, s, X, G = R.gen_layer(0, 64, 8)
    yw = R.svd_fwd_bwd(U, Vv, s, X, G, 8, out_dim=64, in_dim=64)[0]
    p = fb.SvdParam(64, 64, t(U), t(Vv), t(s))
    y, _ = fb.svd_forward(p, t(X), 8)
    e = relative_error(y.double().cpu().numpy(), yw)
    checks.append(("svd layer forward d=64", e <= 1e-4, f"rel {e:.2e}"))
    print(f"{'check':32s} result")
    for name, ok, detail in checks:
        print(f"{name:32s} {'PASS' if ok else 'FAIL'}  {detail}")
    n_ok = sum(ok for _, ok, _ in checks)
    print(f"\n{n_ok}/{len(checks)} checks passed")
    return 0 if n_ok == len(checks) else 2


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description="FastH benchmark (B200): blocked Householder products vs baselines")
    ap.add_argument("--d", default="64,128,256", help="dimensions: comma list or start:step:count")
    ap.add_argument("--m", type=int, default=32, help="mini-batch columns (default 32)")
    ap.add_argument("--k", default="auto", help="block width: integer or 'auto'")
    ap.add_argument("--algo", default="fasth", help="comma list of fasth|ref-fasth|ref-sequential")
    ap.add_argument("--op", default="mul", help="mul|inverse|det|exp|cayley|layer")
    ap.add_argument("--reps", type=int, default=100, help="timed repetitions per record (default 100)")
    ap.add_argument("--seed", type=int, default=0, help="RNG seed")
    ap.add_argument("--threads", type=int, default=0, help="CPU worker count for ref-* (0 = all cores)")
    ap.add_argument("--out", default="", help="CSV output path (default stdout)")
    ap.add_argument("--no-check", dest="check", action="store_false", help="skip the rel_err reference run")
    ap.add_argument("--verify", action="store_true", help="run the verification suite instead of timing")
    try:
        args = ap.parse_args(argv)
        if args.verify:
            return run_verify()
        parse_dims(args.d)
        if args.k != "auto" and not args.k.isdigit():
            raise ValueError("--k: integer or 'auto'")
    except SystemExit as e:
        return 0 if e.code == 0 else 1
    except ValueError as e:
        print(e, file=sys.stderr)
        return 1
    return run(args)


if __name__ == "__main__":
    sys.exit(main())
