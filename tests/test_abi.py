"""CPU checks of the boundary: the C-ABI library loads, exports every symbol
include/fasth_b200.h declares, and fails loudly (no CPU fallback) when no
B200 is present."""
import ctypes as C
import os

import pytest

from paper_2009_13977_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    declared = _lib.header_symbols()
    assert len(declared) >= 25
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    # and every declared symbol has a ctypes signature in the binding
    assert set(declared) <= set(_lib.SIGNATURES)


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib = _lib.load()
    h = C.c_void_p()
    st = lib.fasth_ctx_create(0, None, C.byref(h))
    assert st == 5  # FASTH_ERR_CUDA
    assert b"CUDA" in lib.fasth_last_error() or b"device" in lib.fasth_last_error()
    from paper_2009_13977_b200 import fasth
    with pytest.raises(fasth.Error):
        fasth.fasth_forward(torch.randn(4, 4), torch.randn(4, 2), 2)


def test_status_codes_match_reference_exceptions():
    hdr = open(os.path.join(ROOT, "include", "fasth_b200.h")).read()
    for name, code in (("FASTH_ERR_DIMENSION", 1), ("FASTH_ERR_DEGENERATE", 2),
                       ("FASTH_ERR_SINGULAR", 3), ("FASTH_ERR_INVALID", 4)):
        assert f"{name} = {code}" in hdr
    from paper_2009_13977_b200 import fasth
    assert fasth._ERRORS[1] is fasth.DimensionError
    assert fasth._ERRORS[2] is fasth.DegenerateVectorError
    assert fasth._ERRORS[3] is fasth.SingularMatrixError
