"""Generate tests/golden/fasth_golden.npz from the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    make -C oracle && python tests/golden/make_golden.py

Every array is produced by oracle/_ref/libfasth_ref.so, i.e. the reference
headers compiled as-is behind oracle/ref_shim.cpp, including the reference's
own libstdc++-seeded generators (bench.hpp:74-90, svd_layer.hpp:46-71).  The
fixtures pin both the C restatement (oracle/fasth_oracle.c) and, on the GPU
box where /root/reference is absent, the CUDA path.

Keys are "<case>/<array>"; chains are (n, d), matrices (rows, cols) row-major.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Ref  # noqa: E402


def main():
    R = Ref()
    out: dict[str, np.ndarray] = {}
    meta: dict[str, dict] = {}

    def put(case, info, **arrays):
        meta[case] = info
        for k, v in arrays.items():
            out[f"{case}/{k}"] = np.asarray(v, dtype=np.float64)

    # config 1 of BASELINE.json: Workload(op=mul, seed=0, d=64, m=32), b=8
    V, X, G = R.gen_mul(0, 64, 32)
    Y, dX, dV = R.fasth_fwd_bwd(V, X, G, 8)
    Ys, dXs, dVs = R.sequential_fwd_bwd(V, X, G)
    put("cfg1", {"d": 64, "n": 64, "m": 32, "b": 8, "src": "bench.hpp:117 op=mul seed=0"},
        V=V, X=X, G=G, Y=Y, dX=dX, dV=dV, Y_seq=Ys, dX_seq=dXs, dV_seq=dVs)

    # test_fasth.cpp:95-111: ragged partition d=20 n=17 m=4 b=6 (seed 137 stream)
    V, X, G = R.gen_chain(137, 20, 17, 4)
    Y, dX, dV = R.fasth_fwd_bwd(V, X, G, 6)
    put("ragged", {"d": 20, "n": 17, "m": 4, "b": 6, "src": "test_fasth.cpp:95"},
        V=V, X=X, G=G, Y=Y, dX=dX, dV=dV)

    # edge shapes of acceptance.cpp:58-82: n=1, b=1, b=n, m=1, odd b
    for name, (d, n, m, b, seed) in {"n1": (8, 1, 3, 4, 11), "b1": (16, 16, 8, 1, 12),
                                     "bn": (16, 16, 8, 16, 13), "m1": (64, 64, 1, 8, 14),
                                     "oddb": (64, 32, 32, 7, 15)}.items():
        V, X, G = R.gen_chain(seed, d, n, m)
        Y, dX, dV = R.fasth_fwd_bwd(V, X, G, b)
        put(name, {"d": d, "n": n, "m": m, "b": b, "src": "acceptance.cpp:58-82 shapes"},
            V=V, X=X, G=G, Y=Y, dX=dX, dV=dV)

    # wy.hpp known answers (test_wy.cpp:27-45)
    W, Yw = R.wy_compact(np.array([[3.0, 4.0]]))
    put("kat_wy1", {"src": "test_wy.cpp:27"}, V=np.array([[3.0, 4.0]]), W=W, Y=Yw)
    Vax = np.array([[1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    W, Yw = R.wy_compact(Vax)
    put("kat_wy2", {"src": "test_wy.cpp:36"}, V=Vax, W=W, Y=Yw)
    # householder.hpp reflection KATs (test_dense_core.cpp:26-42)
    put("kat_e1", {"src": "test_dense_core.cpp:26"}, V=np.array([[1.0, 0.0, 0.0]]),
        X=np.eye(3), Y=R.chain_apply(np.array([[1.0, 0.0, 0.0]]), np.eye(3)))
    put("kat_swap", {"src": "test_dense_core.cpp:35"}, V=np.array([[1.0, 1.0]]),
        X=np.array([[1.0], [0.0]]), Y=R.chain_apply(np.array([[1.0, 1.0]]), np.array([[1.0], [0.0]])))

    # a WY block at d=48, b=8 (tape internals)
    V, X, G = R.gen_chain(41, 48, 8, 4)
    W, Yw = R.wy_compact(V)
    put("wy48", {"d": 48, "b": 8, "src": "wy.hpp:56"}, V=V, W=W, Y=Yw)

    # SVD layer (svd_layer.hpp:106-154): square and rectangular (test_svd_layer.cpp:79)
    for name, (o, i, m, b, seed) in {"svd8": (8, 8, 3, 3, 227), "svd6x4": (6, 4, 3, 2, 229),
                                     "svd4x6": (4, 6, 3, 2, 230), "svd64": (64, 64, 16, 8, 231)}.items():
        U, Vv, s, X, G = R.gen_param(seed, o, i, o, i, m)
        Y, dX, dU, dV, ds = R.svd_fwd_bwd(U, Vv, s, X, G, b)
        Uo, Vo, so = R.svd_step(U, Vv, s, dU, dV, ds, 1e-2, 0.5)
        put(name, {"out": o, "in": i, "m": m, "b": b, "eta": 1e-2, "eps": 0.5,
                   "src": "svd_layer.hpp:106-202"},
            U=U, V=Vv, sigma=s, X=X, G=G, Y=Y, dX=dX, dU=dU, dV=dV, dsigma=ds,
            U_step=Uo, V_step=Vo, sigma_step=so)

    # matops (matops.hpp:57-117) at d=32
    U, Vv, s, X, _ = R.gen_layer(5, 32, 4, symmetric=False)
    put("inverse32", {"d": 32, "m": 4, "b": 6, "src": "matops.hpp:69"},
        U=U, V=Vv, sigma=s, X=X, Y=R.matop(0, U, Vv, s, X, 6),
        logdet=np.array([R.log_abs_det(s)]))
    U, Vv, s, X, _ = R.gen_layer(6, 32, 4, symmetric=True)
    put("exp32", {"d": 32, "m": 4, "b": 6, "src": "matops.hpp:98"},
        U=U, sigma=s, X=X, Y=R.matop(1, U, Vv, s, X, 6))
    put("cayley32", {"d": 32, "m": 4, "b": 6, "src": "matops.hpp:107"},
        U=U, sigma=s, X=X, Y=R.matop(2, U, Vv, s, X, 6))

    path = os.path.join(HERE, "fasth_golden.npz")
    np.savez_compressed(path, **out)
    with open(os.path.join(HERE, "fasth_golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
