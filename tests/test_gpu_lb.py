"""Large-batch path (csrc/lb_*.cu): the chain re-blocked into wide WY blocks
on the tcgen05 3xTF32 GEMM.  Checked against a float64 restatement of the
blocked algebra (tests/algo_model.py's, in torch on the GPU so that the
reference-scale shapes finish in milliseconds) and against the chain path."""
import ctypes as C

import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = 1e-4  # north_star: max relative error on UX, dX, dV


def model64(V, X, G, B):
    """tests/algo_model.fwd_bwd in float64 torch.  V: (n, d); X, G: (d, m)."""
    V, X, G = V.double(), X.double(), G.double()
    n, d = V.shape
    Vt = V.t()
    bl = [(lo, min(lo + B, n)) for lo in range(0, n, B)]
    Ts = []
    for lo, hi in bl:
        Vb = Vt[:, lo:hi]
        Gm = Vb.t() @ Vb
        M = torch.diag(torch.diag(Gm)) + 2 * torch.triu(Gm, 1)
        Ts.append(torch.linalg.inv(M))
    A = X.clone()
    acts, zf = [None] * len(bl), [None] * len(bl)
    for i in reversed(range(len(bl))):
        lo, hi = bl[i]
        Vb = Vt[:, lo:hi]
        Zp = Ts[i] @ (Vb.t() @ A)
        A = A - 2 * Vb @ Zp
        acts[i], zf[i] = A, Zp
    Y = A
    Gs = G.clone()
    dV = torch.zeros_like(V)
    for i in range(len(bl)):
        lo, hi = bl[i]
        Vb = Vt[:, lo:hi]
        Zb = Ts[i].t() @ (Vb.t() @ Gs)
        Q = zf[i] @ Zb.t()
        Kp = torch.triu(Q - Q.t(), 1)
        dV[lo:hi] = (-2 * (acts[i] @ Zb.t() + Gs @ zf[i].t() + 2 * Vb @ Kp)).t()
        Gs = Gs - 2 * Vb @ Zb
    return Y, Gs, dV


def rel(a, b):
    return float((a.double() - b).norm() / b.norm())


def inputs(n, d, m, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    V = torch.randn(n, d, device="cuda", generator=g)
    X = torch.randn(m, d, device="cuda", generator=g).t()
    G = torch.randn(m, d, device="cuda", generator=g).t()
    return V, X, G


@pytest.mark.parametrize("n,d,m", [(512, 512, 1024), (1024, 1024, 2048), (384, 256, 640), (2048, 2048, 4096),
                                   (640, 500, 1100), (1536, 1540, 1300), (256, 772, 228), (128, 1024, 4100),
                                   (1024, 1024, 32), (2048, 2048, 128), (512, 1024, 60)])
def test_large_batch_matches_f64(n, d, m, monkeypatch):
    """Small batches included: split K into a reduction epilogue (m < 1024)."""
    from paper_2009_13977_b200 import fasth as fb
    monkeypatch.setenv("FASTH_LB", "1")
    V, X, G = inputs(n, d, m)
    ctx = fb.Context(0)
    n0 = ctx.launch_count
    Y, back = fb.fasth_forward_backward(V, X, G, 32, ctx=ctx)
    torch.cuda.synchronize()
    launches = ctx.launch_count - n0
    Yr, dXr, dVr = model64(V, X, G, 64)
    errs = (rel(Y, Yr), rel(back.grad_input, dXr), rel(back.grad_vectors, dVr))
    print(f"n={n} d={d} m={m}: rel err Y {errs[0]:.2e} dX {errs[1]:.2e} dV {errs[2]:.2e}, {launches} launches")
    assert launches > 10  # the multi-kernel large-batch step ran, not the chain sweep
    assert max(errs) <= TOL, errs


def test_large_batch_agrees_with_chain_path(monkeypatch):
    from paper_2009_13977_b200 import fasth as fb
    V, X, G = inputs(1024, 1024, 1024, seed=3)
    monkeypatch.setenv("FASTH_LB", "1")
    Y1, b1 = fb.fasth_forward_backward(V, X, G, 32)
    monkeypatch.setenv("FASTH_LB", "0")
    Y0, b0 = fb.fasth_forward_backward(V, X, G, 32)
    torch.cuda.synchronize()
    for a, b in ((Y1, Y0), (b1.grad_input, b0.grad_input), (b1.grad_vectors, b0.grad_vectors)):
        assert rel(a, b.double()) <= TOL


def test_large_batch_degenerate_vector_reported(monkeypatch):
    from paper_2009_13977_b200 import fasth as fb
    monkeypatch.setenv("FASTH_LB", "1")
    V, X, G = inputs(512, 512, 1024, seed=5)
    V[300].zero_()
    with pytest.raises(fb.DegenerateVectorError) as ei:
        fb.fasth_forward_backward(V, X, G, 32, ctx=fb.Context(0))
    assert "300" in str(ei.value)


def test_gemm_hook_tcgen05():
    """The GEMM alone (K-major and MN-major B, transposed output, split K)."""
    from paper_2009_13977_b200 import _lib
    lib = _lib.load()
    f = lib.fasthb_lb_gemm_test
    P, I64, I, F = C.c_void_p, C.c_int64, C.c_int, C.c_float
    f.argtypes = [P, I64, P, I64, I, I, I, I, P, I64, F, F, P, I64, P, P, I64, P, P, I64, P, I, I]
    f.restype = I
    p = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None
    g = torch.Generator(device="cuda").manual_seed(1)
    for M, N, K, mn in ((256, 512, 256, 0), (200, 300, 100, 0), (256, 512, 256, 1), (384, 768, 96, 1)):
        A = torch.randn(M, K, device="cuda", generator=g)
        B = torch.randn(K, N, device="cuda", generator=g) if mn else torch.randn(N, K, device="cuda", generator=g)
        Cm = torch.randn(M, N, device="cuda", generator=g)
        ref = -2.0 * (A.double() @ (B.double() if mn else B.double().t())) + Cm.double()
        D = torch.zeros(M, N, device="cuda")
        assert f(p(A), K, p(B), N if mn else K, mn, M, N, K, p(Cm), N, -2.0, 1.0, p(D), N, None, None, N, None,
                 None, M, None, 1, 0) == 0
        assert rel(D, ref) < 1e-5
        Th, Tl = torch.zeros(N, M, device="cuda"), torch.zeros(N, M, device="cuda")
        part = torch.zeros(3, M, N, device="cuda")
        ref2 = A.double() @ (B.double() if mn else B.double().t())
        assert f(p(A), K, p(B), N if mn else K, mn, M, N, K, None, N, 1.0, 0.0, None, N, None, None, N, p(Th),
                 p(Tl), M, None, 1, 0) == 0
        assert rel((Th.double() + Tl.double()).t(), ref2) < 1e-5
        if K >= 96:
            assert f(p(A), K, p(B), N if mn else K, mn, M, N, K, None, N, 1.0, 0.0, None, N, None, None, N, None,
                     None, M, p(part), 3, 0) == 0
            assert rel(part.sum(0), ref2) < 1e-5


def test_large_batch_two_call_equals_fused(monkeypatch):
    """fasth_forward + fasth_backward (tape = the forward stages) run the same
    kernels as the fused call: bitwise equal; the tape is reusable."""
    from paper_2009_13977_b200 import fasth as fb
    monkeypatch.delenv("FASTH_LB", raising=False)  # default selection: m >= 1024, d >= 512
    V, X, G = inputs(1024, 1024, 2048, seed=9)
    Yf, bf = fb.fasth_forward_backward(V, X, G, 32)
    tape = fb.fasth_forward(V, X, 32)
    b1 = fb.fasth_backward(tape, G)
    b2 = fb.fasth_backward(tape, G)
    torch.cuda.synchronize()
    assert torch.equal(tape.output(), Yf)
    for a in (b1, b2):
        assert torch.equal(a.grad_input, bf.grad_input)
        assert torch.equal(a.grad_vectors, bf.grad_vectors)
    Yr, dXr, dVr = model64(V, X, G, 64)
    assert max(rel(Yf, Yr), rel(bf.grad_input, dXr), rel(bf.grad_vectors, dVr)) <= TOL


def test_large_batch_unaligned_outputs(monkeypatch):
    """Output pitches that the 16-byte epilogue stores cannot take go through
    packed temporaries (OutBuf)."""
    from paper_2009_13977_b200 import fasth as fb
    monkeypatch.setenv("FASTH_LB", "1")
    n = d = 512
    m = 1024
    V, X, G = inputs(n, d, m, seed=11)
    Y0, b0 = fb.fasth_forward_backward(V, X, G, 32)
    big = torch.zeros(m, d + 3, device="cuda")  # ld = d + 3
    Y = big[:, :d].t()
    big2 = torch.zeros(m, d + 3, device="cuda")
    dX = big2[:, :d].t()
    dV = torch.empty(n, d, device="cuda")
    fb.fasth_forward_backward(V, X, G, 32, out=(Y, dX, dV))
    torch.cuda.synchronize()
    assert torch.equal(Y, Y0) and torch.equal(dX, b0.grad_input) and torch.equal(dV, b0.grad_vectors)


@pytest.mark.parametrize("M,N,K,b_mn,pair", [(256, 512, 256, 0, 0), (256, 512, 256, 1, 0), (1024, 512, 256, 1, 1),
                                             (512, 768, 96, 0, 1), (300, 200, 64, 1, 0)])
def test_gemm_hook_mn_major_a(M, N, K, b_mn, pair, monkeypatch):
    """A operand stored K x M (MN-major, 32-byte-atom swizzle), 1-CTA and CTA-pair tiles."""
    from paper_2009_13977_b200 import _lib
    if pair:
        monkeypatch.setenv("FASTH_LB_PAIR", "1")
    lib = _lib.load()
    f = lib.fasthb_lb_gemm_test_ex
    P, I64, I, F = C.c_void_p, C.c_int64, C.c_int, C.c_float
    f.argtypes = [P, I64, I, P, I64, I, I, I, I, P, I64, F, F, P, I64, P, P, I64, P, P, I64, P, I, I]
    f.restype = I
    p = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    At = torch.randn(K, M, device="cuda", generator=g)  # A^T stored
    B = torch.randn(K, N, device="cuda", generator=g) if b_mn else torch.randn(N, K, device="cuda", generator=g)
    ref = At.double().t() @ (B.double() if b_mn else B.double().t())
    D = torch.zeros(M, N, device="cuda")
    assert f(p(At), M, 1, p(B), N if b_mn else K, b_mn, M, N, K, None, N, 1.0, 0.0, p(D), N, None, None, N, None,
             None, M, None, 1, 0) == 0
    torch.cuda.synchronize()
    assert rel(D, ref) < 1e-5


def test_large_batch_host_entry_graph(monkeypatch):
    """fasth_forward_backward_host at a large-batch shape: the cached CUDA
    graph captures the two-stream large-batch step (fork/join events) and
    replays it bitwise equal to the device-resident call, call after call."""
    from paper_2009_13977_b200 import fasth as fb
    monkeypatch.delenv("FASTH_LB", raising=False)
    n = d = 512
    m = 1024
    V, X, G = inputs(n, d, m, seed=21)
    Vh = V.cpu().pin_memory()
    Xh = X.t().contiguous().cpu().pin_memory()
    Gh = G.t().contiguous().cpu().pin_memory()
    out = tuple(torch.empty(sh).pin_memory() for sh in ((m, d), (m, d), (n, d)))
    ctx = fb.Context(0)
    Yd, back = fb.fasth_forward_backward(V, X, G, 32, ctx=ctx)
    want = (Yd.t().cpu(), back.grad_input.t().cpu(), back.grad_vectors.cpu())
    for _ in range(3):
        got = fb.forward_backward_host(Vh, Xh, Gh, 32, ctx=ctx, out=out)
        for u, w in zip(got, want):
            assert torch.equal(u, w)


def test_default_selection_mid_batch(monkeypatch):
    """d >= 1024 with m >= 128 takes the re-blocked path by default (it measured
    2.3-5x faster than the panel sweep there); d = 512 stays on the chain kernels."""
    from paper_2009_13977_b200 import fasth as fb
    monkeypatch.delenv("FASTH_LB", raising=False)
    for n, d, m, lb in ((1024, 1024, 128, True), (512, 512, 256, False)):
        V, X, G = inputs(n, d, m, seed=n + m)
        ctx = fb.Context(0)
        ctx.set_timing(True)
        fb.fasth_forward_backward(V, X, G, 32, ctx=ctx)
        names = set(ctx.kernel_times())
        ctx.set_timing(False)
        assert ("large_batch(fwd+bwd)" in names) == lb, names


@pytest.mark.parametrize("count,lb", [(4, True), (2, True), (3, True), (4, False), (0, True)])
def test_dv_bucket_events(count, lb, monkeypatch):
    """fasth_ctx_set_dv_events: each bucket's event fires only once its dV
    rows are final (a side stream copies each slice right after waiting on
    its event; the copies must equal the finished dV), buckets tile [0, n)
    in order, and the chain path reports one whole-dV bucket."""
    from paper_2009_13977_b200 import fasth as fb
    monkeypatch.setenv("FASTH_LB", "1" if lb else "0")
    n = d = 2048 if lb else 256
    m = 1024 if lb else 32
    V, X, G = inputs(n, d, m, seed=11)
    ctx = fb.Context(0)
    ctx.set_dv_buckets(count)
    side = torch.cuda.Stream()
    for rep in range(2):
        dV = torch.full((n, d), float("nan"), device="cuda")
        snap = torch.full((n, d), float("nan"), device="cuda")
        outs = (torch.empty(m, d, device="cuda").t(), torch.empty(m, d, device="cuda").t(), dV)
        fb.fasth_forward_backward(V, X, G, 32, ctx=ctx, out=outs)
        bk = ctx.dv_buckets()
        for lo, hi, ev in bk:
            side.wait_event(ev)
            with torch.cuda.stream(side):
                snap[lo:hi].copy_(dV[lo:hi])
        torch.cuda.synchronize()
        if count == 0:
            assert bk == []
            continue
        want = min(count, n // 512) if lb else 1
        assert len(bk) == want, bk
        assert bk[0][0] == 0 and bk[-1][1] == n and all(a[1] == b[0] for a, b in zip(bk, bk[1:]))
        assert torch.equal(snap, dV), f"rep {rep}: a bucket event fired before its rows were final"
        assert torch.isfinite(dV).all()


def test_dv_buckets_nccl_allreduce_single_rank(monkeypatch):
    """The bench's world > 1 step (sharding.allreduce_dv_buckets on a comm
    stream gated by the bucket events) through a 1-rank NCCL group: runs,
    and the sum over one rank leaves dV unchanged."""
    import socket

    import torch.distributed as dist

    from paper_2009_13977_b200 import fasth as fb
    from paper_2009_13977_b200.sharding import allreduce_dv_buckets
    monkeypatch.setenv("FASTH_LB", "1")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        n = d = 2048
        m = 1024
        V, X, G = inputs(n, d, m, seed=12)
        ctx = fb.Context(0)
        ctx.set_dv_buckets(4)
        comm = torch.cuda.Stream()
        _, ref = fb.fasth_forward_backward(V, X, G, 32, ctx=ctx)
        ref = ref.grad_vectors.clone()
        for _ in range(3):
            _, back = fb.fasth_forward_backward(V, X, G, 32, ctx=ctx)
            allreduce_dv_buckets(back.grad_vectors, ctx.dv_buckets(), comm)
            torch.cuda.current_stream().wait_stream(comm)
        torch.cuda.synchronize()
        assert torch.equal(back.grad_vectors, ref)
    finally:
        dist.destroy_process_group()


def svd_model64(U, V, s, X, G, B=64):
    """The SVD layer (svd_layer.hpp:106-147) in float64 torch on model64:
    T1 = rev(V) chain X, T2 = Sigma T1, Y = U chain T2; backward in reverse."""
    out_dim, in_dim = U.shape[1], V.shape[1]
    k = min(out_dim, in_dim)
    m = X.shape[1]
    Vr = V.flip(0)
    T1, _, _ = model64(Vr, X, torch.zeros_like(X), B)
    T2 = torch.zeros(out_dim, m, dtype=torch.float64, device=X.device)
    T2[:k] = s[:k, None].double() * T1[:k]
    Y, dT2, dU = model64(U, T2, G, B)
    ds = (dT2[:k] * T1[:k]).sum(1)
    dT1 = torch.zeros(in_dim, m, dtype=torch.float64, device=X.device)
    dT1[:k] = s[:k, None].double() * dT2[:k]
    _, dX, dVr = model64(Vr, X, dT1, B)
    return Y, dX, dU, dVr.flip(0), ds


@pytest.mark.parametrize("out_dim,in_dim,m", [(1024, 1024, 1024), (768, 512, 1100), (512, 1024, 1024)])
def test_large_batch_svd_layer(out_dim, in_dim, m, monkeypatch):
    """SVD layer with both legs on the large-batch path (V^T leg on a
    vector-reversed copy of V, Sigma materialised between the legs): the
    two-call, one-call and planned entry points against the float64 model
    and against the chain-kernel layer."""
    from paper_2009_13977_b200 import fasth as fb
    g = torch.Generator(device="cuda").manual_seed(out_dim + in_dim + m)
    U = torch.randn(out_dim, out_dim, device="cuda", generator=g)
    V = torch.randn(in_dim, in_dim, device="cuda", generator=g)
    k = min(out_dim, in_dim)
    s = torch.rand(k, device="cuda", generator=g) * 1.5 + 0.5
    X = torch.randn(m, in_dim, device="cuda", generator=g).t()
    G = torch.randn(m, out_dim, device="cuda", generator=g).t()
    p = fb.SvdParam(out_dim, in_dim, U, V, s)
    want = svd_model64(U, V, s, X, G)

    def grads(gr):
        return (gr.grad_input, gr.grad_U_vectors, gr.grad_V_vectors, gr.grad_sigma)

    monkeypatch.setenv("FASTH_LB", "1")
    ctx = fb.Context(0)
    n0 = ctx.launch_count
    Y1, t1 = fb.svd_forward(p, X, 32, ctx=ctx)
    g1 = fb.svd_backward(p, t1, G)
    launches = ctx.launch_count - n0
    Y2, g2 = fb.svd_forward_backward(p, X, G, 32, ctx=ctx)
    Y3, t3 = fb.svd_forward(p, X, 32, ctx=ctx, plan=fb.svd_plan(p, m, 32, ctx=ctx))
    g3 = fb.svd_backward(p, t3, G)
    monkeypatch.setenv("FASTH_LB", "0")
    Y0, t0 = fb.svd_forward(p, X, 32)
    g0 = fb.svd_backward(p, t0, G)
    torch.cuda.synchronize()
    assert launches > 40, launches  # both legs ran the multi-kernel large-batch step
    got = (Y1,) + grads(g1)
    errs = [rel(a, w) for a, w in zip(got, want)]
    print(f"svd {out_dim}x{in_dim} m={m}: rel err Y/dX/dU/dV/ds " + " ".join(f"{e:.2e}" for e in errs)
          + f", {launches} launches")
    assert max(errs) <= TOL, errs
    for a, b in zip(got, (Y2,) + grads(g2)):
        assert torch.equal(a, b)
    for a, b in zip(got, (Y3,) + grads(g3)):
        assert torch.equal(a, b)
    for a, b in zip(got, (Y0,) + grads(g0)):
        assert rel(a, b.double()) <= TOL


@pytest.mark.parametrize("op", ["inverse", "exponential", "cayley"])
def test_large_batch_sigma_ops(op, monkeypatch):
    """Sigma-ops (matops.hpp:43-117) at large batch: both chain applications
    on the large-batch forward (reversed U^T leg on a reversed copy, f(Sigma)
    rows materialised) against the float64 model and the chain kernels."""
    from paper_2009_13977_b200 import fasth as fb
    d, m = 1024, 2048
    g = torch.Generator(device="cuda").manual_seed(21)
    U = torch.randn(d, d, device="cuda", generator=g)
    s = torch.rand(d, device="cuda", generator=g) * 0.5 + 0.5
    X = torch.randn(m, d, device="cuda", generator=g).t()
    if op == "inverse":
        V = torch.randn(d, d, device="cuda", generator=g)
        fs = 1.0 / s.double()
    else:
        V = torch.empty(0, d, device="cuda")
        fs = torch.exp(s.double()) if op == "exponential" else (1 - s.double()) / (1 + s.double())
    p = fb.SvdParam(d, d, U, V, s)
    fn = getattr(fb, "apply_" + op)
    Z = torch.zeros(d, m, dtype=torch.float64, device="cuda")
    T = model64(U.flip(0), X, Z, 64)[0]
    want = model64(V if op == "inverse" else U, fs[:, None] * T, Z, 64)[0]
    monkeypatch.setenv("FASTH_LB", "1")
    ctx = fb.Context(0)
    n0 = ctx.launch_count
    Y1 = fn(p, X, 32, ctx=ctx)
    launches = ctx.launch_count - n0
    monkeypatch.setenv("FASTH_LB", "0")
    Y0 = fn(p, X, 32, ctx=ctx)
    torch.cuda.synchronize()
    err = rel(Y1, want)
    print(f"{op}: rel err {err:.2e}, {launches} launches")
    assert launches > 20, launches
    assert err <= TOL and rel(Y0, want) <= TOL


def test_dv_buckets_not_reported_for_internal_dv(monkeypatch):
    """Bucket events describe the caller's dV of fasth_backward /
    fasth_forward_backward only: the SVD legs (temporaries) and the host
    entry (dV returned in host memory) report no buckets."""
    from paper_2009_13977_b200 import fasth as fb
    monkeypatch.setenv("FASTH_LB", "1")
    d, m = 512, 1024
    g = torch.Generator(device="cuda").manual_seed(31)
    p = fb.SvdParam(d, d, torch.randn(d, d, device="cuda", generator=g), torch.randn(d, d, device="cuda", generator=g),
                    torch.rand(d, device="cuda", generator=g) + 0.5)
    X = torch.randn(m, d, device="cuda", generator=g).t()
    G = torch.randn(m, d, device="cuda", generator=g).t()
    ctx = fb.Context(0)
    ctx.set_dv_buckets(4)
    fb.fasth_forward_backward(p.V, X, G, 32, ctx=ctx)
    assert len(ctx.dv_buckets()) == 1  # d = 512: one 512-row block
    _, t = fb.svd_forward(p, X, 32, ctx=ctx)
    fb.svd_backward(p, t, G)
    torch.cuda.synchronize()
    assert ctx.dv_buckets() == []
    Vh, Xh, Gh = p.V.cpu().pin_memory(), X.t().contiguous().cpu().pin_memory(), G.t().contiguous().cpu().pin_memory()
    fb.forward_backward_host(Vh, Xh, Gh, 32, ctx=ctx)
    assert ctx.dv_buckets() == []


def test_large_batch_without_dx(monkeypatch):
    """dX not requested (NULL through the C ABI): the last gradient update is
    skipped; Y and dV unchanged bit for bit."""
    from paper_2009_13977_b200 import fasth as fb
    monkeypatch.setenv("FASTH_LB", "1")
    n = d = 1024
    m = 1024
    V, X, G = inputs(n, d, m, seed=41)
    ctx = fb.Context(0)
    Y0, b0 = fb.fasth_forward_backward(V, X, G, 32, ctx=ctx)
    Y1 = torch.empty(m, d, device="cuda").t()
    dV1 = torch.empty(n, d, device="cuda")
    P = C.c_void_p
    rc = ctx.lib.fasth_forward_backward(ctx.h, P(V.data_ptr()), d, d, n, P(X.data_ptr()), d, P(G.data_ptr()), d, m,
                                        32, P(Y1.data_ptr()), d, None, d, P(dV1.data_ptr()), d)
    torch.cuda.synchronize()
    assert rc == 0
    assert torch.equal(Y0, Y1) and torch.equal(b0.grad_vectors, dV1)
