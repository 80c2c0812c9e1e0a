"""OSVD checkpoint files (svd_layer.hpp:204-290): the format, pinned to files
the unmodified reference wrote (tests/golden/make_osvd.py), and the device
load / save path of the C ABI (fasth_svd_load / fasth_svd_save)."""
import os
import struct

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


def parse_osvd(path):
    """Plain restatement of load_svd_param (svd_layer.hpp:254-273)."""
    raw = open(path, "rb").read()
    assert raw[:4] == b"OSVD"
    version, out_dim, in_dim, nu, nv = struct.unpack("<5I", raw[4:24])
    assert version == 1
    vals = np.frombuffer(raw[24:], dtype="<f8")
    k = min(out_dim, in_dim)
    assert vals.size == nu * out_dim + nv * in_dim + k
    U = vals[:nu * out_dim].reshape(nu, out_dim)
    V = vals[nu * out_dim:nu * out_dim + nv * in_dim].reshape(nv, in_dim)
    return out_dim, in_dim, U, V, vals[-k:]


def test_reference_files_parse_to_their_arrays():
    g = np.load(os.path.join(GOLD, "osvd_golden.npz"))
    for name, pre in (("osvd_ref_6x4.bin", "ref"), ("osvd_f32_5x7.bin", "f32")):
        out_dim, in_dim, U, V, s = parse_osvd(os.path.join(GOLD, name))
        assert np.array_equal(U, g[f"{pre}_U"]) and np.array_equal(V, g[f"{pre}_V"])
        assert np.array_equal(s, g[f"{pre}_s"])


def test_header_info_without_gpu():
    from paper_2009_13977_b200 import fasth as fb
    assert fb.svd_file_info(os.path.join(GOLD, "osvd_ref_6x4.bin")) == (6, 4, 6, 4)
    assert fb.svd_file_info(os.path.join(GOLD, "osvd_f32_5x7.bin")) == (5, 7, 5, 3)


def test_header_errors_match_reference(tmp_path):
    from paper_2009_13977_b200 import fasth as fb
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"XSVD" + bytes(20))
    with pytest.raises(fb.Error, match="bad magic"):
        fb.svd_file_info(str(bad))
    bad.write_bytes(b"OSVD" + struct.pack("<I", 2) + bytes(16))
    with pytest.raises(fb.Error, match="unsupported version"):
        fb.svd_file_info(str(bad))
    bad.write_bytes(b"OSVD" + struct.pack("<2I", 1, 3))
    with pytest.raises(fb.Error, match="truncated header"):
        fb.svd_file_info(str(bad))


@pytest.mark.gpu
def test_device_load_save_round_trip(tmp_path):
    from paper_2009_13977_b200 import fasth as fb
    g = np.load(os.path.join(GOLD, "osvd_golden.npz"))
    p = fb.load_svd_param_file(os.path.join(GOLD, "osvd_ref_6x4.bin"))
    assert (p.out_dim, p.in_dim) == (6, 4)
    assert np.allclose(p.U.double().cpu().numpy(), g["ref_U"], rtol=1e-7, atol=1e-7)
    assert np.allclose(p.V.double().cpu().numpy(), g["ref_V"], rtol=1e-7, atol=1e-7)
    assert np.allclose(p.sigma.double().cpu().numpy(), g["ref_s"], rtol=1e-7)
    # fp32-representable payload: device load + save reproduces the reference file bit for bit
    src = os.path.join(GOLD, "osvd_f32_5x7.bin")
    out = tmp_path / "rt.bin"
    fb.save_svd_param_file(fb.load_svd_param_file(src), str(out))
    assert out.read_bytes() == open(src, "rb").read()


@pytest.mark.gpu
def test_device_save_loads_in_reference(tmp_path):
    from paper_2009_13977_b200 import fasth as fb
    try:
        from oracle.oracle import Ref
        R = Ref()
    except Exception:
        pytest.skip("oracle/_ref not built")
    import torch
    U = torch.randn(3, 5, device="cuda")
    V = torch.randn(2, 5, device="cuda")
    s = torch.rand(5, device="cuda") + 0.5
    path = tmp_path / "dev.bin"
    fb.save_svd_param_file(fb.SvdParam(5, 5, U, V, s), str(path))
    out_dim, in_dim, Ur, Vr, sr = R.svd_load(str(path))
    assert (out_dim, in_dim) == (5, 5)
    assert np.array_equal(Ur, U.double().cpu().numpy()) and np.array_equal(Vr, V.double().cpu().numpy())
    assert np.array_equal(sr, s.double().cpu().numpy())


@pytest.mark.gpu
def test_device_load_rejects_degenerate_vector(tmp_path):
    from paper_2009_13977_b200 import fasth as fb
    raw = bytearray(open(os.path.join(GOLD, "osvd_ref_6x4.bin"), "rb").read())
    raw[24 + 6 * 8:24 + 12 * 8] = bytes(48)  # U vector 1 -> zero
    path = tmp_path / "deg.bin"
    path.write_bytes(bytes(raw))
    with pytest.raises(fb.DegenerateVectorError):
        fb.load_svd_param_file(str(path))
    path.write_bytes(bytes(raw[:60]))
    with pytest.raises(fb.Error, match="truncated payload"):
        fb.load_svd_param_file(str(path))


@pytest.mark.gpu
def test_tune_block_width():
    from paper_2009_13977_b200 import fasth as fb
    assert fb.tune_block_width(784, 32) == 28  # round(sqrt(784)), fasth.hpp:149-152
    b = fb.tune_block_width(128, 16, timed=True)
    assert 2 <= b <= 2 * 12 or b == 16
    assert fb.tune_block_width(128, 16, timed=True) == b  # cached
