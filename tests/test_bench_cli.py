"""tools/fasth_bench_b200.py: the reference CLI's flag and record contract
(tools/fasth_bench.cpp:23-42, 81-90; bench.hpp:67)."""
import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, os.path.join(ROOT, "tools"))

import fasth_bench_b200 as cli  # noqa: E402


def test_parse_dims_like_reference():
    assert cli.parse_dims("64,128,256") == [64, 128, 256]
    assert cli.parse_dims("64:64:4") == [64, 128, 192, 256]
    with pytest.raises(ValueError, match="start:step:count"):
        cli.parse_dims("64:64")


def test_configuration_errors_exit_1():
    assert cli.main(["--d", "64:x:2"]) == 1
    assert cli.main(["--k", "fast"]) == 1
    assert cli.main(["--bogus-flag"]) == 1


def test_header_extends_reference_schema():
    ref = "algo,op,d,m,k,reps,threads,mean_s,std_s"
    assert cli.HEADER.startswith(ref)
    assert cli.HEADER.split(",")[len(ref.split(",")):] == ["rel_err", "gpus", "tflops", "roofline_frac"]


@pytest.mark.gpu
def test_cli_records_and_verify(tmp_path):
    out = tmp_path / "r.csv"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fasth_bench_b200.py"), "--d", "64,128",
                        "--m", "16", "--k", "8", "--reps", "3", "--op", "mul", "--out", str(out)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = out.read_text().strip().splitlines()
    assert lines[0] == cli.HEADER and len(lines) == 3
    for ln in lines[1:]:
        f = ln.split(",")
        assert f[0] == "fasth" and float(f[7]) > 0 and float(f[9]) <= 1e-4
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fasth_bench_b200.py"), "--d", "64",
                        "--m", "8", "--k", "8", "--reps", "2", "--op", "inverse"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    assert float(r.stdout.strip().splitlines()[1].split(",")[9]) <= 1e-4
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fasth_bench_b200.py"), "--verify"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "checks passed" in r.stdout
