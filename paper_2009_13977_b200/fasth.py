"""Python mirror of the reference FastH API over the C ABI.

Same names, argument meaning and error behaviour as the reference's
header-only C++ API (/root/reference/proj/include/fasth/), with torch CUDA
tensors in place of ``fasth::Matrix``:

=====================================  ==========================================
reference (file:line)                  here
=====================================  ==========================================
``fasth_forward`` fasth.hpp:40         ``fasth_forward(V, X, block_width)``
``fasth_backward`` fasth.hpp:69        ``fasth_backward(tape, G)``
``svd_forward`` svd_layer.hpp:106      ``svd_forward(p, X, block_width)``
``svd_backward`` svd_layer.hpp:122     ``svd_backward(p, tape, G)``
``svd_step`` svd_layer.hpp:158         ``svd_step(p, grads, eta)``
``clamp_sigma`` svd_layer.hpp:196      ``clamp_sigma(p, epsilon)``
``apply_inverse`` matops.hpp:69        ``apply_inverse(p, X, block_width)``
``apply_exponential`` matops.hpp:98    ``apply_exponential(p, X, block_width)``
``apply_cayley`` matops.hpp:107        ``apply_cayley(p, X, block_width)``
``log_abs_det`` matops.hpp:57          ``log_abs_det(p)``
``apply_pseudo_inverse`` matops.hpp:158 ``apply_pseudo_inverse(p, X, tol, bw)``
``wy_compact`` wy.hpp:56               ``wy_compact(vectors)``
``wy_apply`` wy.hpp:104                ``wy_apply(block, X)``
``wy_apply_transpose`` wy.hpp:137      ``wy_apply_transpose(block, X)``
``compact_chain`` wy.hpp:151           ``compact_chain(V, block_width)``
``TapeForward::compacted`` /           ``Tape.compacted`` / ``Tape.activations``
``::activations`` fasth.hpp:22-29      (materialised on first access)
=====================================  ==========================================

Shapes follow the reference: a chain is an ``(n, d)`` tensor (row k = v_k,
chain order), activations are ``(d, m)`` (rows = dimension, columns = batch).
Activations are stored column-major on the device (each sample contiguous);
inputs in any layout are accepted, outputs are ``(d, m)`` views of
column-major storage.  All arithmetic runs in the sm_100a kernels of
``lib/libfasth_b200.so``; nothing here computes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib

# ---- error hierarchy (matrix.hpp:12-30) -----------------------------------


class Error(RuntimeError):
    """fasth::Error"""


class DimensionError(Error):
    """fasth::DimensionError"""


class DegenerateVectorError(Error):
    """fasth::DegenerateVectorError"""


class SingularMatrixError(Error):
    """fasth::SingularMatrixError"""


class CudaError(Error):
    pass


_ERRORS = {1: DimensionError, 2: DegenerateVectorError, 3: SingularMatrixError, 4: Error,
           5: CudaError, 6: CudaError}


def _check(status: int):
    if status:
        msg = _lib.load().fasth_last_error().decode()
        raise _ERRORS.get(status, Error)(msg)


# ---- context -------------------------------------------------------------


class Context:
    """One per (device, stream).  ``stream=None`` follows torch's current
    stream at every call.  ``deferred=True`` latches device-side errors
    (degeneracy, singular sigma) until :meth:`check` instead of
    synchronising inside each call."""

    def __init__(self, device: int = 0, deferred: bool = False):
        self.lib = _lib.load()
        self.device = device
        h = C.c_void_p()
        with torch.cuda.device(device):
            _check(self.lib.fasth_ctx_create(device, None, C.byref(h)))
        self.h = h
        self.set_deferred(deferred)

    def set_deferred(self, deferred: bool):
        _check(self.lib.fasth_ctx_set_check(self.h, 1 if deferred else 0))
        self.deferred = deferred

    def bind_stream(self, stream: torch.cuda.Stream | None = None):
        s = stream if stream is not None else torch.cuda.current_stream(self.device)
        _check(self.lib.fasth_ctx_set_stream(self.h, C.c_void_p(s.cuda_stream)))

    def check(self):
        _check(self.lib.fasth_ctx_check(self.h))

    def set_timing(self, on, graph: bool = False):
        """Per-kernel CUDA-event timing.  graph=True keeps the events alive so
        a CUDA graph captured while timing is on can be replayed and read with
        kernel_times() after every replay (no host gaps in the figures)."""
        _check(self.lib.fasth_ctx_set_timing(self.h, (2 if graph else 1) if on else 0))

    def kernel_times(self) -> dict:
        """{kernel: (total_ms, launches)} accumulated in timing mode."""
        buf = C.create_string_buffer(1 << 16)
        self.lib.fasth_ctx_kernel_times(self.h, buf, len(buf))
        out = {}
        for line in buf.value.decode().splitlines():
            name, ms, cnt = line.rsplit(" ", 2)
            out[name] = (float(ms), int(cnt))
        return out

    def set_dv_buckets(self, count: int):
        """Ask later fasth_backward / fasth_forward_backward calls to signal
        dV row buckets as they complete (fasth_ctx_set_dv_events): ``count``
        torch CUDA events, read back with :meth:`dv_buckets`.  0 turns it off."""
        evs = [torch.cuda.Event() for _ in range(count)]
        with torch.cuda.device(self.device):
            for e in evs:  # torch creates the CUDA event on first record
                e.record()
        arr = (C.c_void_p * max(count, 1))(*[C.c_void_p(e.cuda_event) for e in evs])
        _check(self.lib.fasth_ctx_set_dv_events(self.h, arr, count))
        self._dv_events = evs

    def dv_buckets(self) -> list:
        """[(row_begin, row_end, event)] of the last call's dV buckets, in
        completion order; all-reduce dV[row_begin:row_end] on a stream that
        waits on `event`."""
        evs = getattr(self, "_dv_events", [])
        ends = (C.c_int64 * max(len(evs), 1))()
        k = self.lib.fasth_ctx_dv_buckets(self.h, ends, len(evs))
        out, lo = [], 0
        for i in range(max(k, 0)):
            out.append((lo, int(ends[i]), evs[i]))
            lo = int(ends[i])
        return out

    @property
    def launch_count(self) -> int:
        return int(self.lib.fasth_ctx_launch_count(self.h))

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.fasth_ctx_destroy(self.h)
                self.h = None
        except Exception:
            pass


_default: dict[int, Context] = {}


def default_context(device: int | None = None) -> Context:
    dev = torch.cuda.current_device() if device is None else device
    if dev not in _default:
        _default[dev] = Context(dev)
    return _default[dev]


def _ctx(ctx, t: torch.Tensor) -> Context:
    c = ctx if ctx is not None else default_context(t.device.index)
    c.bind_stream()
    return c


# ---- layout helpers --------------------------------------------------------


def _dev_f32(t: torch.Tensor, what: str) -> torch.Tensor:
    if not isinstance(t, torch.Tensor):
        raise Error(f"{what}: expected a torch tensor")
    if not t.is_cuda:
        raise Error(f"{what}: expected a CUDA tensor (no CPU path)")
    if t.dtype != torch.float32:
        t = t.float()
    return t


def _colmajor(X: torch.Tensor, what: str):
    """(d, m) tensor -> (tensor, ld) with column-major storage."""
    X = _dev_f32(X, what)
    if X.dim() != 2:
        raise DimensionError(f"{what}: expected a 2-D (d, m) tensor")
    d, m = X.shape
    if X.stride(0) == 1 and (m <= 1 or X.stride(1) >= max(d, 1)):
        return X, max(X.stride(1), d, 1)
    Xc = X.t().contiguous().t()
    return Xc, max(d, 1)


def _chain(V: torch.Tensor, what: str, d: int | None = None):
    """(n, d) chain tensor -> (tensor, n, d, ld) as column-major d x n."""
    V = _dev_f32(V, what)
    if V.dim() != 2:
        raise DimensionError(f"{what}: expected an (n, d) chain tensor")
    n, dd = V.shape
    if d is not None and n > 0 and dd != d:
        raise DimensionError(f"{what}: vector length {dd} != dim {d}")
    if n > 0 and not (V.stride(1) == 1 and V.stride(0) >= dd):
        V = V.contiguous()
    return V, n, (dd if n > 0 or d is None else d), max(V.stride(0) if n > 0 else dd, 1)


def _new_out(d: int, m: int, like: torch.Tensor) -> torch.Tensor:
    return torch.empty((m, d), dtype=torch.float32, device=like.device).t()


def _out_ld(T, d: int, m: int, what: str) -> int:
    """Leading dimension of a caller-provided (d, m) output with column-major storage."""
    if T is None:
        return max(d, 1)
    if tuple(T.shape) != (d, m) or (m > 1 and d > 1 and T.stride(0) != 1):
        raise DimensionError(f"out {what}: expected a column-major ({d}, {m}) tensor")
    return max(T.stride(1) if m > 1 else d, d, 1)


def _check_out(T, like: torch.Tensor, what: str) -> torch.Tensor:
    """A caller-provided output: float32 on the input's device (shape and
    column-major layout are checked by _out_ld)."""
    if not isinstance(T, torch.Tensor) or T.dtype != torch.float32 or T.device != like.device:
        raise Error(f"out {what}: expected a float32 tensor on {like.device}")
    return T


def _host_f32(T, shape, what: str) -> torch.Tensor:
    """A host buffer of the host-buffer entry: CPU float32, C-contiguous, the
    given shape (the C ABI reads and writes it through raw pointers)."""
    if not isinstance(T, torch.Tensor) or T.is_cuda or T.dtype != torch.float32 or not T.is_contiguous() \
            or tuple(T.shape) != tuple(shape):
        raise DimensionError(f"forward_backward_host: {what} must be a contiguous CPU float32 tensor of shape "
                             f"{tuple(shape)}")
    return T


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None and t.numel() > 0 else None


# ---- FastH (fasth.hpp) ------------------------------------------------------


@dataclass
class WYBlock:
    """WYBlock (wy.hpp:18-25): I - 2 W Y^T = H_1 ... H_width.  W and Y are
    (dim, width) views of column-major device storage; source_vectors is the
    (width, dim) slice of the chain."""
    dim: int
    width: int
    W: torch.Tensor
    Y: torch.Tensor
    source_vectors: torch.Tensor
    sequential_steps: int = 0


@dataclass
class CompactedChain:
    """CompactedChain (wy.hpp:29-48)."""
    dim: int
    block_width: int
    blocks: list

    def factor_count(self) -> int:
        return sum(b.width for b in self.blocks)

    def compaction_stages(self) -> int:
        return max((b.sequential_steps for b in self.blocks), default=0)


def _blocks(V, W, Y, d, n, bw):
    return [WYBlock(d, min(bw, n - lo), W[lo:lo + bw].t(), Y[lo:lo + bw].t(), V[lo:lo + bw],
                    min(bw, n - lo)) for lo in range(0, n, bw)]


def compact_chain(V: torch.Tensor, block_width: int, *, ctx: Context | None = None) -> CompactedChain:
    """wy.hpp:151 — the chain (n, d) as ceil(n / block_width) WY blocks (the last ragged)."""
    V, n, d, ldv = _chain(V, "compact_chain: V")
    if not 1 <= int(block_width) <= n:
        raise Error(f"compact_chain: block width {block_width} outside [1, {n}]")
    c = _ctx(ctx, V)
    W = torch.empty((n, d), dtype=torch.float32, device=V.device)
    Y = torch.empty((n, d), dtype=torch.float32, device=V.device)
    _check(c.lib.fasth_compact_chain(c.h, _ptr(V), ldv, d, n, int(block_width), _ptr(W), d, _ptr(Y), d))
    return CompactedChain(d, int(block_width), _blocks(V, W, Y, d, n, int(block_width)))


def wy_compact(vectors: torch.Tensor, *, ctx: Context | None = None) -> WYBlock:
    """wy.hpp:56 — (W, Y) of the b >= 1 vectors (rows of ``vectors``)."""
    if vectors.dim() != 2 or vectors.shape[0] == 0:
        raise Error("wy_compact: empty vector list")
    V, n, d, ldv = _chain(vectors, "wy_compact: vectors")
    c = _ctx(ctx, V)
    W = torch.empty((n, d), dtype=torch.float32, device=V.device)
    Y = torch.empty((n, d), dtype=torch.float32, device=V.device)
    _check(c.lib.fasth_wy_compact(c.h, _ptr(V), ldv, d, n, _ptr(W), d, _ptr(Y), d))
    return _blocks(V, W, Y, d, n, n)[0]


def _wy_apply(fn, block: WYBlock, X, ctx, out=None):
    X, ldx = _colmajor(X, fn)
    d, m = X.shape
    if d != block.dim:
        raise DimensionError(f"{fn}: X has {d} rows, block dim {block.dim}")
    c = _ctx(ctx, X)
    W, ldw = _colmajor(block.W, fn)
    Y, ldy = _colmajor(block.Y, fn)
    O = _new_out(d, m, X) if out is None else out
    _check(getattr(c.lib, "fasth_" + fn)(c.h, _ptr(W), ldw, _ptr(Y), ldy, d, block.width, _ptr(X), ldx, m,
                                          _ptr(O), _out_ld(O, d, m, "out")))
    return O


def wy_apply(block: WYBlock, X: torch.Tensor, *, ctx: Context | None = None) -> torch.Tensor:
    """wy.hpp:104 — X - 2 W (Y^T X)."""
    return _wy_apply("wy_apply", block, X, ctx)


def wy_apply_transpose(block: WYBlock, X: torch.Tensor, *, ctx: Context | None = None) -> torch.Tensor:
    """wy.hpp:137 — X - 2 Y (W^T X)."""
    return _wy_apply("wy_apply_transpose", block, X, ctx)


class Tape:
    """TapeForward (fasth.hpp:22-29): the device record the backward runs
    from, plus the reference's members ``compacted`` (the WY blocks) and
    ``activations`` (A_1..A_{q+1}: ``activations[q]`` is X, ``[0]`` the
    output), materialised on first access by compact_chain and the block
    recurrence A_i = wy_apply(P_i, A_{i+1}) (fasth.hpp:55-59)."""

    def __init__(self, ctx: Context, handle, output: torch.Tensor, d: int, n: int, m: int, b: int,
                 V: torch.Tensor | None = None, X: torch.Tensor | None = None):
        self.ctx, self.h = ctx, handle
        self._output = output
        self.d, self.n, self.m, self.block_width = d, n, m, b
        self._V, self._X = V, X
        self._compacted = self._activations = None

    def output(self) -> torch.Tensor:
        return self._output

    def input(self) -> torch.Tensor:
        return self._X

    def _materialise(self):
        if self._compacted is not None:
            return
        if self._X is None:
            raise Error("Tape: recorded without its input (record=False)")
        bw = min(max(self.block_width, 1), max(self.n, 1))
        if self.n == 0:
            self._compacted = CompactedChain(self.d, self.block_width, [])
            self._activations = [self._X]
            return
        cc = compact_chain(self._V, bw, ctx=self.ctx)
        acts = [None] * (len(cc.blocks) + 1)
        acts[-1] = self._X
        for i in reversed(range(len(cc.blocks))):
            acts[i] = wy_apply(cc.blocks[i], acts[i + 1], ctx=self.ctx)
        self._compacted, self._activations = cc, acts

    @property
    def compacted(self) -> CompactedChain:
        self._materialise()
        return self._compacted

    @property
    def activations(self) -> list:
        self._materialise()
        return self._activations

    def block_count(self) -> int:
        q = C.c_int()
        _check(self.ctx.lib.fasth_tape_info(self.h, None, None, None, None, C.byref(q)))
        return q.value

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.ctx.lib.fasth_tape_destroy(self.h)
                self.h = None
        except Exception:
            pass


@dataclass
class BackwardResult:
    """BackwardResult (fasth.hpp:31-34); grad_vectors is (n, d)."""
    grad_input: torch.Tensor
    grad_vectors: torch.Tensor


def fasth_forward(V: torch.Tensor, X: torch.Tensor, block_width: int, *, ctx: Context | None = None,
                  record: bool = True, out: torch.Tensor | None = None) -> Tape:
    """fasth.hpp:40 — returns a Tape whose ``output()`` is H_1...H_n X."""
    X, ldx = _colmajor(X, "fasth_forward: X")
    d, m = X.shape
    V, n, dv, ldv = _chain(V, "fasth_forward: V", d)
    if n > 0 and dv != d:
        raise DimensionError("fasth_forward: X row count != chain dim")
    c = _ctx(ctx, X)
    Y = _new_out(d, m, X) if out is None else _check_out(out, X, "Y")
    ldy = _out_ld(Y, d, m, "Y")
    h = C.c_void_p()
    _check(c.lib.fasth_forward(c.h, _ptr(V), ldv, d, n, _ptr(X), ldx, m, int(block_width),
                               _ptr(Y), ldy, C.byref(h) if record else None))
    return Tape(c, h if record else None, Y, d, n, m, int(block_width), V, X)


def fasth_backward(tape: Tape, G: torch.Tensor, *, want_vectors: bool = True) -> BackwardResult:
    """fasth.hpp:69 — dX = U^T G and the Eq. (5) gradients of every vector."""
    if tape.h is None:
        raise Error("fasth_backward: tape was recorded with record=False")
    G, ldg = _colmajor(G, "fasth_backward: grad_output")
    if tuple(G.shape) != (tape.d, tape.m):
        raise DimensionError("fasth_backward: grad_output shape mismatch")
    c = tape.ctx
    c.bind_stream()
    dX = _new_out(tape.d, tape.m, G)
    dV = torch.empty((tape.n, tape.d), dtype=torch.float32, device=G.device) if want_vectors else None
    _check(c.lib.fasth_backward(c.h, tape.h, _ptr(G), ldg, _ptr(dX), max(tape.d, 1),
                                _ptr(dV), max(tape.d, 1)))
    return BackwardResult(dX, dV)


def fasth_forward_backward(V: torch.Tensor, X: torch.Tensor, G: torch.Tensor, block_width: int, *,
                           ctx: Context | None = None, want_vectors: bool = True, out=None):
    """fasth.hpp:40 + :69 as one call (``fasth_forward_backward``), for a
    caller that already holds grad_output G (the reference benchmark's
    op=mul step, bench.hpp:147-151).  Returns (Y, BackwardResult)."""
    X, ldx = _colmajor(X, "fasth_forward: X")
    G, ldg = _colmajor(G, "fasth_backward: grad_output")
    d, m = X.shape
    if tuple(G.shape) != (d, m):
        raise DimensionError("fasth_backward: grad_output shape mismatch")
    V, n, dv, ldv = _chain(V, "fasth_forward: V", d)
    if n > 0 and dv != d:
        raise DimensionError("fasth_forward: X row count != chain dim")
    c = _ctx(ctx, X)
    if out is None:
        Y, dX = _new_out(d, m, X), _new_out(d, m, X)
        dV = torch.empty((n, d), dtype=torch.float32, device=X.device) if want_vectors else None
    else:
        Y, dX, dV = out
    ldy, lddx = _out_ld(Y, d, m, "Y"), _out_ld(dX, d, m, "dX")
    lddv = max(dV.stride(0), d, 1) if dV is not None and dV.dim() == 2 and dV.stride(1) == 1 else max(d, 1)
    _check(c.lib.fasth_forward_backward(c.h, _ptr(V), ldv, d, n, _ptr(X), ldx, _ptr(G), ldg, m,
                                        int(block_width), _ptr(Y), ldy, _ptr(dX), lddx,
                                        _ptr(dV), lddv))
    return Y, BackwardResult(dX, dV)


def forward_backward_host(V, X, G, block_width: int, *, ctx: Context | None = None, out=None):
    """Host-buffer drop-in for fasth_forward + fasth_backward
    (``fasth_forward_backward_host``).  V: (n, d), X, G: (m, d) CPU float32
    tensors (pin them for full bandwidth) — i.e. column-major d x m.
    Returns (Y, dX, dV) as CPU tensors of the same layouts; ``out`` may hold
    preallocated (pinned) ones."""
    c = ctx if ctx is not None else default_context()
    c.bind_stream()
    if not isinstance(V, torch.Tensor) or V.dim() != 2 or not isinstance(X, torch.Tensor) or X.dim() != 2:
        raise DimensionError("forward_backward_host: V must be (n, d) and X (m, d)")
    n, d = V.shape
    m = X.shape[0]
    _host_f32(V, (n, d), "V")
    _host_f32(X, (m, d), "X")
    _host_f32(G, (m, d), "G")
    if out is None:
        Y = torch.empty((m, d), dtype=torch.float32, pin_memory=True)
        dX = torch.empty((m, d), dtype=torch.float32, pin_memory=True)
        dV = torch.empty((n, d), dtype=torch.float32, pin_memory=True)
    else:
        Y, dX, dV = (_host_f32(t, sh, w) for t, sh, w in zip(out, ((m, d), (m, d), (n, d)), ("Y", "dX", "dV")))
    _check(c.lib.fasth_forward_backward_host(c.h, _ptr(V), d, n, _ptr(X), _ptr(G), m,
                                             int(block_width), _ptr(Y), _ptr(dX), _ptr(dV)))
    return Y, dX, dV


# ---- SVD layer (svd_layer.hpp) ---------------------------------------------


@dataclass
class SvdParam:
    """SvdParam (svd_layer.hpp:25-72): U (nu, out_dim), V (nv, in_dim),
    sigma (min(out_dim, in_dim),)."""
    out_dim: int
    in_dim: int
    U: torch.Tensor
    V: torch.Tensor
    sigma: torch.Tensor

    def min_dim(self) -> int:
        return min(self.out_dim, self.in_dim)

    def validate(self):
        if self.U.shape[0] and self.U.shape[1] != self.out_dim or \
                self.V.shape[0] and self.V.shape[1] != self.in_dim:
            raise DimensionError("SvdParam: chain dims inconsistent")
        if self.sigma.numel() != self.min_dim():
            raise DimensionError("SvdParam: sigma length != min(out_dim, in_dim)")

    def _c(self) -> _lib.SvdParamC:
        self.validate()
        self.U = _dev_f32(self.U, "SvdParam.U").contiguous()
        self.V = _dev_f32(self.V, "SvdParam.V").contiguous()
        self.sigma = _dev_f32(self.sigma, "SvdParam.sigma").contiguous()
        return _lib.SvdParamC(self.out_dim, self.in_dim, self.U.shape[0], self.V.shape[0],
                              _ptr(self.U), self.out_dim, _ptr(self.V), self.in_dim,
                              _ptr(self.sigma))


@dataclass
class SvdGradients:
    """SvdGradients (svd_layer.hpp:74-79)."""
    grad_U_vectors: torch.Tensor
    grad_V_vectors: torch.Tensor
    grad_sigma: torch.Tensor
    grad_input: torch.Tensor


class SvdTape:
    """SvdTape (svd_layer.hpp:83-86), opaque."""

    def __init__(self, ctx, handle, m):
        self.ctx, self.h, self.m = ctx, handle, m

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.ctx.lib.fasth_svd_tape_destroy(self.h)
                self.h = None
        except Exception:
            pass


class SvdPlan:
    """Both legs' WY blocks built ahead of a forward (``fasth_svd_plan_create``);
    single use: ``svd_forward(..., plan=)`` consumes it."""

    def __init__(self, ctx, handle, m, block_width):
        self.ctx, self.h, self.m, self.block_width = ctx, handle, m, block_width

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.ctx.lib.fasth_svd_plan_destroy(self.h)
                self.h = None
        except Exception:
            pass


def svd_plan(p: SvdParam, m: int, block_width: int, *, side_stream: bool = True,
             ctx: Context | None = None) -> SvdPlan:
    """Build layer p's WY blocks now (on the context's side stream by default),
    for a later ``svd_forward(p, X, block_width, plan=...)`` with X of m columns."""
    pc = p._c()
    c = _ctx(ctx, p.sigma)
    h = C.c_void_p()
    _check(c.lib.fasth_svd_plan_create(c.h, C.byref(pc), int(m), int(block_width), int(side_stream), C.byref(h)))
    return SvdPlan(c, h, m, block_width)


def svd_forward(p: SvdParam, X: torch.Tensor, block_width: int, *, ctx: Context | None = None,
                plan: SvdPlan | None = None):
    """svd_layer.hpp:106 — returns (Y, tape), Y = U (Sigma (V^T X)).  With
    ``plan`` (from ``svd_plan``) the prepared WY blocks are used (and consumed)."""
    X, ldx = _colmajor(X, "svd_forward: X")
    if X.shape[0] != p.in_dim:
        raise DimensionError(f"svd_forward: X has {X.shape[0]} rows, in_dim {p.in_dim}")
    pc = p._c()
    c = _ctx(ctx, X)
    m = X.shape[1]
    Y = _new_out(p.out_dim, m, X)
    h = C.c_void_p()
    if plan is not None:
        if not plan.h:
            raise Error("svd_forward: plan already consumed")
        _check(c.lib.fasth_svd_forward_planned(c.h, C.byref(pc), plan.h, _ptr(X), ldx, m, int(block_width),
                                               _ptr(Y), max(p.out_dim, 1), C.byref(h)))
    else:
        _check(c.lib.fasth_svd_forward(c.h, C.byref(pc), _ptr(X), ldx, m, int(block_width), _ptr(Y),
                                       max(p.out_dim, 1), C.byref(h)))
    return Y, SvdTape(c, h, m)


def svd_backward(p: SvdParam, tape: SvdTape, G: torch.Tensor) -> SvdGradients:
    """svd_layer.hpp:122."""
    G, ldg = _colmajor(G, "svd_backward: grad_output")
    if tuple(G.shape) != (p.out_dim, tape.m):
        raise DimensionError("svd_backward: grad_output shape mismatch")
    pc = p._c()
    c = tape.ctx
    c.bind_stream()
    dev = G.device
    dX = _new_out(p.in_dim, tape.m, G)
    dU = torch.empty((p.U.shape[0], p.out_dim), dtype=torch.float32, device=dev)
    dV = torch.empty((p.V.shape[0], p.in_dim), dtype=torch.float32, device=dev)
    ds = torch.empty(p.min_dim(), dtype=torch.float32, device=dev)
    _check(c.lib.fasth_svd_backward(c.h, C.byref(pc), tape.h, _ptr(G), ldg, _ptr(dX),
                                    max(p.in_dim, 1), _ptr(dU), max(p.out_dim, 1), _ptr(dV),
                                    max(p.in_dim, 1), _ptr(ds)))
    return SvdGradients(dU, dV, ds, dX)


def svd_forward_backward(p: SvdParam, X: torch.Tensor, G: torch.Tensor, block_width: int, *,
                         ctx: Context | None = None):
    """svd_forward + svd_backward in one call (``fasth_svd_forward_backward``)
    for a caller holding grad_output up front (bench.hpp:166-209's layer
    step).  Returns (Y, SvdGradients)."""
    X, ldx = _colmajor(X, "svd_forward: X")
    G, ldg = _colmajor(G, "svd_backward: grad_output")
    if X.shape[0] != p.in_dim or tuple(G.shape) != (p.out_dim, X.shape[1]):
        raise DimensionError("svd_forward_backward: X / grad_output shape mismatch")
    pc = p._c()
    c = _ctx(ctx, X)
    m = X.shape[1]
    dev = X.device
    Y = _new_out(p.out_dim, m, X)
    dX = _new_out(p.in_dim, m, X)
    dU = torch.empty((p.U.shape[0], p.out_dim), dtype=torch.float32, device=dev)
    dV = torch.empty((p.V.shape[0], p.in_dim), dtype=torch.float32, device=dev)
    ds = torch.empty(p.min_dim(), dtype=torch.float32, device=dev)
    _check(c.lib.fasth_svd_forward_backward(c.h, C.byref(pc), _ptr(X), ldx, _ptr(G), ldg, m, int(block_width),
                                            _ptr(Y), max(p.out_dim, 1), _ptr(dX), max(p.in_dim, 1), _ptr(dU),
                                            max(p.out_dim, 1), _ptr(dV), max(p.in_dim, 1), _ptr(ds)))
    return Y, SvdGradients(dU, dV, ds, dX)


def svd_step(p: SvdParam, g: SvdGradients, eta: float, *, clamp_epsilon: float | None = None,
             inplace: bool = False, ctx: Context | None = None) -> SvdParam:
    """svd_layer.hpp:158 (optionally fused with clamp_sigma, :196).

    The reference's svd_step is pure (it returns a new SvdParam and rejects a
    degenerate update before anything changes).  ``inplace=True`` writes the
    update into ``p`` itself, so a degeneracy error raised by the step leaves
    ``p`` already updated; use the default (a new parameter) where that
    matters."""
    if clamp_epsilon is not None and not (0.0 <= float(clamp_epsilon) < 1.0):
        raise Error("clamp_sigma: epsilon outside [0, 1)")
    pc = p._c()
    if g.grad_U_vectors.shape != p.U.shape or g.grad_V_vectors.shape != p.V.shape or \
            g.grad_sigma.numel() != p.sigma.numel():
        raise DimensionError("svd_step: gradient shapes do not match parameter")
    c = _ctx(ctx, p.sigma)
    out = p if inplace else SvdParam(p.out_dim, p.in_dim, torch.empty_like(p.U),
                                     torch.empty_like(p.V), torch.empty_like(p.sigma))
    dU = g.grad_U_vectors.contiguous()
    dV = g.grad_V_vectors.contiguous()
    _check(c.lib.fasth_svd_step(c.h, C.byref(pc), _ptr(dU), max(p.out_dim, 1), _ptr(dV),
                                max(p.in_dim, 1), _ptr(g.grad_sigma.contiguous()), float(eta),
                                -1.0 if clamp_epsilon is None else float(clamp_epsilon),
                                _ptr(out.U), max(p.out_dim, 1), _ptr(out.V), max(p.in_dim, 1),
                                _ptr(out.sigma)))
    return out


def clamp_sigma(p: SvdParam, epsilon: float, *, ctx: Context | None = None) -> SvdParam:
    """svd_layer.hpp:196."""
    c = _ctx(ctx, p.sigma)
    s = _dev_f32(p.sigma, "sigma").contiguous()
    out = torch.empty_like(s)
    _check(c.lib.fasth_clamp_sigma(c.h, _ptr(s), s.numel(), float(epsilon), _ptr(out)))
    return SvdParam(p.out_dim, p.in_dim, p.U, p.V, out)


def _sigma_op(fn_name, p: SvdParam, X, block_width, ctx):
    X, ldx = _colmajor(X, fn_name)
    pc = p._c()
    c = _ctx(ctx, X)
    d, m = X.shape
    Y = _new_out(d, m, X)
    _check(getattr(c.lib, fn_name)(c.h, C.byref(pc), _ptr(X), ldx, m, int(block_width), _ptr(Y),
                                   max(d, 1)))
    return Y


def apply_inverse(p: SvdParam, X, block_width: int, *, ctx=None):
    """matops.hpp:69 — W^{-1} X = V Sigma^{-1} U^T X."""
    return _sigma_op("fasth_apply_inverse", p, X, block_width, ctx)


def apply_exponential(p: SvdParam, X, block_width: int, *, ctx=None):
    """matops.hpp:98 — e^W X for the symmetric form (empty V chain)."""
    return _sigma_op("fasth_apply_exponential", p, X, block_width, ctx)


def apply_cayley(p: SvdParam, X, block_width: int, *, ctx=None):
    """matops.hpp:107 — (I - W)(I + W)^{-1} X for the symmetric form."""
    return _sigma_op("fasth_apply_cayley", p, X, block_width, ctx)


def apply_pseudo_inverse(p: SvdParam, X, tol: float, block_width: int, *, ctx=None):
    """matops.hpp:158 — W^+ X = V Sigma^+ U^T X (rectangular allowed: X is
    (out_dim, m), the result (in_dim, m))."""
    if tol < 0:
        raise Error("apply_pseudo_inverse: negative tolerance")
    X, ldx = _colmajor(X, "apply_pseudo_inverse")
    if X.shape[0] != p.out_dim:
        raise DimensionError("apply_pseudo_inverse: X row count mismatch")
    pc = p._c()
    c = _ctx(ctx, X)
    m = X.shape[1]
    Y = _new_out(p.in_dim, m, X)
    _check(c.lib.fasth_apply_pseudo_inverse(c.h, C.byref(pc), _ptr(X), ldx, m, float(tol), int(block_width), _ptr(Y),
                                            max(p.in_dim, 1)))
    return Y


def log_abs_det(p: SvdParam, *, ctx=None) -> float:
    """matops.hpp:57 — sum ln|sigma_i| (square parameters)."""
    pc = p._c()
    c = _ctx(ctx, p.sigma)
    out = C.c_double()
    _check(c.lib.fasth_log_abs_det(c.h, C.byref(pc), C.byref(out)))
    return out.value


# ---- OSVD checkpoints (svd_layer.hpp:204-290) -----------------------------


def svd_file_info(path: str) -> tuple[int, int, int, int]:
    """(out_dim, in_dim, nU, nV) of an OSVD file (header only)."""
    h = [C.c_int() for _ in range(4)]
    _check(_lib.load().fasth_svd_file_info(str(path).encode(), *[C.byref(x) for x in h]))
    return tuple(x.value for x in h)


def load_svd_param_file(path: str, *, device: int | None = None, ctx: Context | None = None) -> SvdParam:
    """svd_layer.hpp:282 — the checkpoint straight into device buffers (fp32)."""
    out_dim, in_dim, nu, nv = svd_file_info(path)
    c = ctx if ctx is not None else default_context(device)
    c.bind_stream()
    dev = torch.device("cuda", c.device)
    U = torch.empty((nu, out_dim), dtype=torch.float32, device=dev)
    V = torch.empty((nv, in_dim), dtype=torch.float32, device=dev)
    sigma = torch.empty((min(out_dim, in_dim),), dtype=torch.float32, device=dev)
    _check(c.lib.fasth_svd_load(c.h, str(path).encode(), _ptr(U), out_dim, _ptr(V), in_dim, _ptr(sigma)))
    return SvdParam(out_dim, in_dim, U, V, sigma)


def save_svd_param_file(p: SvdParam, path: str, *, ctx: Context | None = None):
    """svd_layer.hpp:276 — the device parameter written as the reference's f64 OSVD file."""
    pc = p._c()
    c = _ctx(ctx, p.sigma)
    _check(c.lib.fasth_svd_save(c.h, C.byref(pc), str(path).encode()))


def tune_block_width(d: int, m: int, timed: bool = False, seed: int = 0x5EED, *,
                     ctx: Context | None = None) -> int:
    """fasth.hpp:147 — analytic round(sqrt(d)), or the fastest block width of a
    timed search on the device (cached per (d, m))."""
    c = ctx if ctx is not None else default_context()
    c.bind_stream()
    out = C.c_int()
    _check(c.lib.fasth_tune_block_width(c.h, int(d), int(m), 1 if timed else 0, int(seed), C.byref(out)))
    return out.value
