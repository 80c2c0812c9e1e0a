"""TEST INFRASTRUCTURE ONLY — numpy front end of the CPU oracle.

Two back ends, both f64 and both CPU-only:

* ``Port`` — ``oracle/_build/liboracle.so``, the plain-C restatement in
  ``oracle/fasth_oracle.c`` (every function cites the reference lines it
  follows).
* ``Ref`` — ``oracle/_ref/libfasth_ref.so``, the UNMODIFIED reference headers
  (``/root/reference/proj/include/fasth``) compiled by ``oracle/Makefile``
  behind the ``extern "C"`` shim ``oracle/ref_shim.cpp``.  It also exposes the
  reference's own seeded generators (libstdc++ ``mt19937_64`` +
  ``normal_distribution``) so the GPU path sees the reference's exact inputs,
  and ``bench::run_bench`` for the CPU baseline.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline /
``--impl reference``) may import this module, and only as the checker.

Array conventions: a chain is ``(n, d)`` (row k = v_k, chain order); a matrix
is ``(rows, cols)`` C-order, exactly the reference ``Matrix`` (matrix.hpp:66).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libfasth_ref.so")
REF_NATIVE_SO = os.path.join(HERE, "_ref", "libfasth_ref_native.so")


def _native_ok() -> bool:
    """The -march=native build runs here iff this CPU has the ISA extensions
    of the CPU it was compiled on (AVX-512 / AMX of Sapphire Rapids class)."""
    try:
        flags = set(open("/proc/cpuinfo").read().split("flags", 2)[1].split("\n", 1)[0].split())
    except Exception:
        return False
    march = ""
    try:
        march = open(os.path.join(HERE, "_ref", "native_march.txt")).read().strip()
    except Exception:
        pass
    need = {"avx512f", "avx512bw", "avx512vl", "avx512_fp16", "amx_tile"} if march in (
        "sapphirerapids", "emeraldrapids", "graniterapids") else {"__unknown__"}
    return need <= flags


def ref_so_path() -> str:
    return REF_NATIVE_SO if os.path.exists(REF_NATIVE_SO) and _native_ok() else REF_SO

_D = C.POINTER(C.c_double)
_SZ = C.c_size_t


class OracleError(RuntimeError):
    """Mirrors the reference's error hierarchy by status code."""

    KINDS = {1: "DimensionError", 2: "DegenerateVectorError", 3: "SingularMatrixError",
             4: "Error", 5: "Error"}

    def __init__(self, code: int, msg: str = ""):
        self.code = code
        self.kind = self.KINDS.get(code, "Error")
        super().__init__(f"{self.kind}: {msg}")


def _p(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_D)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def build():
    """Compile the oracle libraries (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class Port:
    """The C restatement (oracle/fasth_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)

    def _chk(self, rc):
        if rc:
            raise OracleError(rc)

    def chain_apply(self, V, X):
        V, X = _f64(V), _f64(X)
        n, d = V.shape if V.size else (0, X.shape[0])
        Y = np.empty_like(X)
        self._chk(self.lib.orc_chain_apply(_SZ(d), _SZ(n), _SZ(X.shape[1]), _p(V), _p(X), _p(Y)))
        return Y

    def householder_grad(self, v, A, G):
        v, A, G = _f64(v), _f64(A), _f64(G)
        out = np.empty_like(v)
        self._chk(self.lib.orc_householder_grad(_SZ(v.size), _SZ(A.shape[1]), _p(v), _p(A),
                                                _p(G), _p(out)))
        return out

    def sequential_fwd_bwd(self, V, X, G):
        V, X, G = _f64(V), _f64(X), _f64(G)
        d, m = X.shape
        n = V.shape[0]
        Y, dX, dV = np.empty_like(X), np.empty_like(X), np.empty((n, d))
        self._chk(self.lib.orc_sequential_fwd_bwd(_SZ(d), _SZ(n), _SZ(m), _p(V), _p(X), _p(G),
                                                  _p(Y), _p(dX), _p(dV)))
        return Y, dX, dV

    def wy_compact(self, V):
        V = _f64(V)
        b, d = V.shape
        W, Y = np.empty((b, d)), np.empty((b, d))
        self._chk(self.lib.orc_wy_compact(_SZ(d), _SZ(b), _p(V), _p(W), _p(Y)))
        return W, Y

    def fasth_fwd_bwd(self, V, X, G, b):
        V, X = _f64(V), _f64(X)
        d, m = X.shape
        n = V.shape[0]
        Y = np.empty_like(X)
        if G is None:
            self._chk(self.lib.orc_fasth_fwd_bwd(_SZ(d), _SZ(n), _SZ(m), _SZ(b), _p(V), _p(X),
                                                 None, _p(Y), None, None))
            return Y
        G = _f64(G)
        dX, dV = np.empty_like(X), np.empty((n, d))
        self._chk(self.lib.orc_fasth_fwd_bwd(_SZ(d), _SZ(n), _SZ(m), _SZ(b), _p(V), _p(X), _p(G),
                                             _p(Y), _p(dX), _p(dV)))
        return Y, dX, dV

    def svd_fwd_bwd(self, U, V, sigma, X, G, b, out_dim=None, in_dim=None):
        U, V, sigma, X = _f64(U), _f64(V), _f64(sigma), _f64(X)
        in_dim = X.shape[0] if in_dim is None else in_dim
        out_dim = (U.shape[1] if U.size else len(sigma)) if out_dim is None else out_dim
        m = X.shape[1]
        nu, nv = U.shape[0], V.shape[0]
        Y = np.empty((out_dim, m))
        if G is None:
            self._chk(self.lib.orc_svd_fwd_bwd(_SZ(out_dim), _SZ(in_dim), _SZ(nu), _SZ(nv), _SZ(m),
                                               _SZ(b), _p(U), _p(V), _p(sigma), _p(X), None,
                                               _p(Y), None, None, None, None))
            return Y
        G = _f64(G)
        dX, dU, dV = np.empty((in_dim, m)), np.empty((nu, out_dim)), np.empty((nv, in_dim))
        ds = np.empty(min(out_dim, in_dim))
        self._chk(self.lib.orc_svd_fwd_bwd(_SZ(out_dim), _SZ(in_dim), _SZ(nu), _SZ(nv), _SZ(m),
                                           _SZ(b), _p(U), _p(V), _p(sigma), _p(X), _p(G), _p(Y),
                                           _p(dX), _p(dU), _p(dV), _p(ds)))
        return Y, dX, dU, dV, ds

    def svd_step(self, U, V, sigma, dU, dV, ds, eta, clamp_eps=-1.0, out_dim=None, in_dim=None):
        U, V, sigma, dU, dV, ds = map(_f64, (U, V, sigma, dU, dV, ds))
        out_dim = U.shape[1] if out_dim is None else out_dim
        in_dim = V.shape[1] if in_dim is None else in_dim
        Uo, Vo, so = np.empty_like(U), np.empty_like(V), np.empty_like(sigma)
        bc, bi = C.c_int(-1), C.c_long(-1)
        rc = self.lib.orc_svd_step(_SZ(out_dim), _SZ(in_dim), _SZ(U.shape[0]), _SZ(V.shape[0]),
                                   _p(U), _p(V), _p(sigma), _p(dU), _p(dV), _p(ds),
                                   C.c_double(eta), C.c_double(clamp_eps), _p(Uo), _p(Vo), _p(so),
                                   C.byref(bc), C.byref(bi))
        if rc:
            raise OracleError(rc, f"chain {'UV'[bc.value] if bc.value >= 0 else '?'} vector {bi.value}")
        return Uo, Vo, so

    def matop(self, kind, U, V, sigma, X, b):
        U, V, sigma, X = map(_f64, (U, V, sigma, X))
        d, m = X.shape
        Y = np.empty_like(X)
        self._chk(self.lib.orc_matop(C.c_int(kind), _SZ(d), _SZ(U.shape[0]), _SZ(V.shape[0]),
                                     _SZ(m), _SZ(b), _p(U), _p(V), _p(sigma), _p(X), _p(Y)))
        return Y

    def log_abs_det(self, sigma):
        sigma = _f64(sigma)
        out = C.c_double()
        self._chk(self.lib.orc_log_abs_det(_SZ(sigma.size), _p(sigma), C.byref(out)))
        return out.value


class Ref:
    """The unmodified reference compiled behind oracle/ref_shim.cpp."""

    def __init__(self, path: str | None = None):
        if path is None:
            if not os.path.exists(REF_SO):
                build()
            path = ref_so_path()
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: build it where /root/reference exists")
        self.path = path
        self.march = "native" if path == REF_NATIVE_SO else "x86-64-v3"
        self.lib = C.CDLL(path)
        self.lib.ref_last_error.restype = C.c_char_p

    def _chk(self, rc):
        if rc:
            raise OracleError(rc, self.lib.ref_last_error().decode())

    def hardware_threads(self) -> int:
        return int(self.lib.ref_hardware_threads())

    # ---- the reference's own seeded generators ---------------------------
    def gen_mul(self, seed, d, m):
        """bench.hpp:117-134, op=mul: (V n=d x d, X d x m, G d x m)."""
        V, X, G = np.empty((d, d)), np.empty((d, m)), np.empty((d, m))
        self._chk(self.lib.ref_gen_mul(C.c_uint64(seed), _SZ(d), _SZ(m), _p(V), _p(X), _p(G)))
        return V, X, G

    def gen_layer(self, seed, d, m, symmetric=False):
        """bench.hpp:122-134 for op=layer/det/inverse (symmetric=False) or exp/cayley."""
        U, V, s = np.empty((d, d)), np.empty((0 if symmetric else d, d)), np.empty(d)
        X, G = np.empty((d, m)), np.empty((d, m))
        Vp = _p(V) if V.size else None
        self._chk(self.lib.ref_gen_layer(C.c_uint64(seed), _SZ(d), _SZ(m), C.c_int(int(symmetric)),
                                         _p(U), Vp, _p(s), _p(X), _p(G)))
        return U, V, s, X, G

    def gen_chain(self, seed, d, n, m):
        V, X, G = np.empty((n, d)), np.empty((d, m)), np.empty((d, m))
        self._chk(self.lib.ref_gen_chain(C.c_uint64(seed), _SZ(d), _SZ(n), _SZ(m), _p(V) if n else None,
                                         _p(X), _p(G)))
        return V, X, G

    def gen_param(self, seed, out_dim, in_dim, nu, nv, m, lo=0.5, hi=2.0):
        U, V = np.empty((nu, out_dim)), np.empty((nv, in_dim))
        s = np.empty(min(out_dim, in_dim))
        X, G = np.empty((in_dim, m)), np.empty((out_dim, m))
        self._chk(self.lib.ref_gen_param(C.c_uint64(seed), _SZ(out_dim), _SZ(in_dim), _SZ(nu),
                                         _SZ(nv), _SZ(m), C.c_double(lo), C.c_double(hi),
                                         _p(U) if nu else None, _p(V) if nv else None, _p(s),
                                         _p(X), _p(G)))
        return U, V, s, X, G

    # ---- OSVD files (svd_layer.hpp:204-290) ---------------------------------
    def svd_save(self, path, U, V, sigma, out_dim, in_dim):
        U, V, s = _f64(U), _f64(V), _f64(sigma)
        self._chk(self.lib.ref_svd_save(str(path).encode(), _SZ(out_dim), _SZ(in_dim), _SZ(U.shape[0]),
                                        _SZ(V.shape[0]), _p(U) if U.size else None, _p(V) if V.size else None,
                                        _p(s)))

    def svd_load(self, path):
        dims = (C.c_size_t * 4)()
        self._chk(self.lib.ref_svd_load(str(path).encode(), dims, None, None, None))
        out_dim, in_dim, nu, nv = (int(x) for x in dims)
        U, V, s = np.empty((nu, out_dim)), np.empty((nv, in_dim)), np.empty(min(out_dim, in_dim))
        self._chk(self.lib.ref_svd_load(str(path).encode(), dims, _p(U) if nu else None, _p(V) if nv else None,
                                        _p(s)))
        return out_dim, in_dim, U, V, s

    # ---- algorithms -------------------------------------------------------
    def fasth_fwd_bwd(self, V, X, G, b):
        V, X = _f64(V), _f64(X)
        d, m = X.shape
        n = V.shape[0]
        Y = np.empty_like(X)
        if G is None:
            self._chk(self.lib.ref_fasth_fwd_bwd(_SZ(d), _SZ(n), _SZ(m), _SZ(b), _p(V), _p(X),
                                                 None, _p(Y), None, None))
            return Y
        G = _f64(G)
        dX, dV = np.empty_like(X), np.empty((n, d))
        self._chk(self.lib.ref_fasth_fwd_bwd(_SZ(d), _SZ(n), _SZ(m), _SZ(b), _p(V), _p(X), _p(G),
                                             _p(Y), _p(dX), _p(dV)))
        return Y, dX, dV

    def fasth_tape(self, V, X, b):
        V, X = _f64(V), _f64(X)
        d, m = X.shape
        n = V.shape[0]
        bb = min(max(b, 1), n)
        q = -(-n // bb)
        act = np.empty((q + 1, d, m))
        W, Y = np.empty((n, d)), np.empty((n, d))
        self._chk(self.lib.ref_fasth_tape(_SZ(d), _SZ(n), _SZ(m), _SZ(b), _p(V), _p(X), _p(act),
                                          _p(W), _p(Y)))
        return act, W, Y

    def sequential_fwd_bwd(self, V, X, G):
        V, X, G = _f64(V), _f64(X), _f64(G)
        d, m = X.shape
        n = V.shape[0]
        Y, dX, dV = np.empty_like(X), np.empty_like(X), np.empty((n, d))
        self._chk(self.lib.ref_sequential_fwd_bwd(_SZ(d), _SZ(n), _SZ(m), _p(V), _p(X), _p(G),
                                                  _p(Y), _p(dX), _p(dV)))
        return Y, dX, dV

    def chain_apply(self, V, X):
        V, X = _f64(V), _f64(X)
        d, m = X.shape
        Y = np.empty_like(X)
        self._chk(self.lib.ref_chain_apply(_SZ(d), _SZ(V.shape[0]), _SZ(m), _p(V) if V.size else None,
                                           _p(X), _p(Y)))
        return Y

    def wy_compact(self, V):
        V = _f64(V)
        b, d = V.shape
        W, Y = np.empty((b, d)), np.empty((b, d))
        self._chk(self.lib.ref_wy_compact(_SZ(d), _SZ(b), _p(V), _p(W), _p(Y)))
        return W, Y

    def householder_grad(self, v, A, G):
        v, A, G = _f64(v), _f64(A), _f64(G)
        out = np.empty_like(v)
        self._chk(self.lib.ref_householder_grad(_SZ(v.size), _SZ(A.shape[1]), _p(v), _p(A), _p(G),
                                                _p(out)))
        return out

    def svd_fwd_bwd(self, U, V, sigma, X, G, b, out_dim=None, in_dim=None):
        U, V, sigma, X = _f64(U), _f64(V), _f64(sigma), _f64(X)
        in_dim = X.shape[0] if in_dim is None else in_dim
        out_dim = (U.shape[1] if U.size else len(sigma)) if out_dim is None else out_dim
        m = X.shape[1]
        nu, nv = U.shape[0], V.shape[0]
        Y = np.empty((out_dim, m))
        Up, Vp = (_p(U) if nu else None), (_p(V) if nv else None)
        if G is None:
            self._chk(self.lib.ref_svd_fwd_bwd(_SZ(out_dim), _SZ(in_dim), _SZ(nu), _SZ(nv), _SZ(m),
                                               _SZ(b), Up, Vp, _p(sigma), _p(X), None, _p(Y),
                                               None, None, None, None))
            return Y
        G = _f64(G)
        dX, dU, dV = np.empty((in_dim, m)), np.empty((nu, out_dim)), np.empty((nv, in_dim))
        ds = np.empty(min(out_dim, in_dim))
        self._chk(self.lib.ref_svd_fwd_bwd(_SZ(out_dim), _SZ(in_dim), _SZ(nu), _SZ(nv), _SZ(m),
                                           _SZ(b), Up, Vp, _p(sigma), _p(X), _p(G), _p(Y), _p(dX),
                                           _p(dU) if nu else None, _p(dV) if nv else None, _p(ds)))
        return Y, dX, dU, dV, ds

    def svd_step(self, U, V, sigma, dU, dV, ds, eta, clamp_eps=-1.0, out_dim=None, in_dim=None):
        U, V, sigma, dU, dV, ds = map(_f64, (U, V, sigma, dU, dV, ds))
        out_dim = U.shape[1] if out_dim is None else out_dim
        in_dim = V.shape[1] if in_dim is None else in_dim
        Uo, Vo, so = np.empty_like(U), np.empty_like(V), np.empty_like(sigma)
        self._chk(self.lib.ref_svd_step(_SZ(out_dim), _SZ(in_dim), _SZ(U.shape[0]), _SZ(V.shape[0]),
                                        _p(U), _p(V), _p(sigma), _p(dU), _p(dV), _p(ds),
                                        C.c_double(eta), C.c_double(clamp_eps), _p(Uo), _p(Vo),
                                        _p(so)))
        return Uo, Vo, so

    def matop(self, kind, U, V, sigma, X, b):
        U, V, sigma, X = map(_f64, (U, V, sigma, X))
        d, m = X.shape
        Y = np.empty_like(X)
        self._chk(self.lib.ref_matop(C.c_int(kind), _SZ(d), _SZ(U.shape[0]), _SZ(V.shape[0]), _SZ(m),
                                     _SZ(b), _p(U) if U.size else None, _p(V) if V.size else None,
                                     _p(sigma), _p(X), _p(Y)))
        return Y

    def pinv(self, U, V, sigma, X, tol, b, out_dim, in_dim):
        """apply_pseudo_inverse (matops.hpp:158): X (out_dim, m) -> (in_dim, m)."""
        U, V, sigma, X = map(_f64, (U, V, sigma, X))
        Y = np.empty((in_dim, X.shape[1]))
        self._chk(self.lib.ref_pinv(_SZ(out_dim), _SZ(in_dim), _SZ(U.shape[0]), _SZ(V.shape[0]), _SZ(X.shape[1]),
                                    _SZ(b), C.c_double(tol), _p(U) if U.size else None, _p(V) if V.size else None,
                                    _p(sigma), _p(X), _p(Y)))
        return Y

    def log_abs_det(self, sigma):
        sigma = _f64(sigma)
        out = C.c_double()
        self._chk(self.lib.ref_log_abs_det(_SZ(sigma.size), _p(sigma), C.byref(out)))
        return out.value

    def run_bench(self, op, algo, d, m, k, reps, seed=0, threads=0):
        """bench::run_bench (bench.hpp:225) for one algorithm: (mean_s, std_s, k)."""
        mean, std, ku = C.c_double(), C.c_double(), C.c_size_t()
        self._chk(self.lib.ref_run_bench(op.encode(), algo.encode(), _SZ(d), _SZ(m), _SZ(k),
                                         _SZ(reps), C.c_uint64(seed), C.c_int(threads),
                                         C.byref(mean), C.byref(std), C.byref(ku)))
        return mean.value, std.value, ku.value

    def verify(self):
        p, t = C.c_int(), C.c_int()
        self._chk(self.lib.ref_verify(C.byref(p), C.byref(t)))
        return p.value, t.value


def relative_error(a, b) -> float:
    """matrix.hpp:106-110: ||a - b||_F / max(||b||_F, 1)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1.0))


def flops_fwd_bwd(d, n, m, b) -> float:
    """F_alg = 12 d n m + 4 d n b (useful fp32 flops)."""
    return 12.0 * d * n * m + 4.0 * d * n * b
