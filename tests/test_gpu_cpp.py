"""The C++ drop-in (include/fasth_b200.hpp) against the unmodified reference
headers, in one binary (tests/cpp/test_dropin.cpp): same seeded inputs through
`fasth::` (CPU f64) and `fasth_b200::` (B200), relative_error <= 1e-4."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "_bin", "test_dropin")


def test_cpp_dropin_matches_reference():
    assert os.path.exists(BIN), "build with `make -C tests/cpp` where the reference tree exists"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "ALL PASSED" in r.stdout
