"""The reference's public WY internals (wy.hpp:56-170) and TapeForward's
members (fasth.hpp:22-29) through the Python mirror, against the reference
compiled as-is (oracle/_ref): compact_chain's W and Y in the reference's
layout, wy_apply / wy_apply_transpose, and the tape's activations with the
block recurrence of test_fasth.cpp:39-50 holding bitwise."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def fb():
    from paper_2009_13977_b200 import fasth
    return fasth


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import Ref
    return Ref()


def dev(a):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def host(t):
    return t.detach().double().cpu().numpy()


def rel(a, b):
    from oracle.oracle import relative_error
    return relative_error(host(a) if not isinstance(a, np.ndarray) else a, b)


@pytest.mark.parametrize("d,n,b", [(96, 70, 16), (784, 784, 32), (12, 12, 5), (33, 7, 7), (64, 64, 1)])
def test_tape_members_match_reference(fb, ref, d, n, b):
    rng = np.random.default_rng(d + n + b)
    V, X = rng.standard_normal((n, d)), rng.standard_normal((d, 3))
    acts, Wc, Yc = ref.fasth_tape(V, X, b)
    tape = fb.fasth_forward(dev(V), dev(X), b)
    q = -(-n // b)
    assert len(tape.activations) == q + 1 and len(tape.compacted.blocks) == q
    assert tape.compacted.factor_count() == n
    W = np.concatenate([host(blk.W).T for blk in tape.compacted.blocks])
    Y = np.concatenate([host(blk.Y).T for blk in tape.compacted.blocks])
    assert rel(W, Wc) <= 1e-5 and rel(Y, Yc) <= 1e-5
    assert max(rel(a, acts[i]) for i, a in enumerate(tape.activations)) <= TOL
    assert rel(tape.output(), acts[0]) <= TOL
    # test_fasth.cpp:39-50: the recurrence holds exactly on the materialised members
    for i, blk in enumerate(tape.compacted.blocks):
        again = fb.wy_apply(blk, tape.activations[i + 1])
        assert np.array_equal(host(again), host(tape.activations[i]))


def test_wy_compact_and_apply_vs_reference(fb, ref):
    rng = np.random.default_rng(47)
    V, X = rng.standard_normal((8, 32)), rng.standard_normal((32, 4))
    W, Y = ref.wy_compact(V)
    blk = fb.wy_compact(dev(V))
    assert blk.width == 8 and blk.dim == 32 and blk.sequential_steps == 8
    assert rel(host(blk.W).T, W) <= 1e-5 and rel(host(blk.Y).T, Y) <= 1e-5
    assert rel(fb.wy_apply(blk, dev(X)), ref.chain_apply(V, X)) <= 1e-5
    # P^T P = I and the transpose of the dense block
    assert rel(fb.wy_apply_transpose(blk, fb.wy_apply(blk, dev(X))), X) <= 1e-5
    import torch
    eye = torch.eye(32, device="cuda")
    assert rel(fb.wy_apply_transpose(blk, eye), host(fb.wy_apply(blk, eye)).T) <= 1e-6
    # single factor: W = Y = v / ||v|| (test_wy.cpp:27-35)
    one = fb.wy_compact(dev(np.array([[3.0, 4.0]])))
    assert np.allclose(host(one.W)[:, 0], [0.6, 0.8]) and np.allclose(host(one.Y)[:, 0], [0.6, 0.8])
    zero = fb.wy_apply(one, torch.zeros(2, 3, device="cuda"))
    assert not host(zero).any()


def test_wy_errors(fb):
    import torch
    with pytest.raises(fb.Error):
        fb.wy_compact(torch.empty(0, 4, device="cuda"))
    V = torch.randn(8, 8, device="cuda")
    for bw in (0, 9):
        with pytest.raises(fb.Error):
            fb.compact_chain(V, bw)
    cc = fb.compact_chain(V, 3)
    assert [b.width for b in cc.blocks] == [3, 3, 2]
    assert all(torch.equal(b.source_vectors, V[3 * i:3 * i + b.width]) for i, b in enumerate(cc.blocks))
    with pytest.raises(fb.DimensionError):
        fb.wy_apply(cc.blocks[0], torch.randn(5, 2, device="cuda"))
    bad = V.clone()
    bad[4] = 0
    with pytest.raises(fb.DegenerateVectorError):
        fb.compact_chain(bad, 3)
