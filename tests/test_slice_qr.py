"""The factored slice cost (paper_2407_20713_b200/csrc/slice_qr.hpp) on the
host: the binary128 Householder factor of random market grids of 1..600
quotes, evaluated as the kernels do (nine FMAs), against the per-quote sum of
calibration.cpp:253-267 in x86 long double (tools/slice_qr_check.cpp).  It
must be as accurate as the reference's own per-quote arithmetic in double,
including rank-deficient grids (n < 4) and near-perfect fits."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
def test_factored_slice_cost_accuracy(tmp_path):
    exe = tmp_path / "slice_qr_check"
    csrc = os.path.join(ROOT, "paper_2407_20713_b200", "csrc")
    subprocess.run(["g++", "-O2", "-std=c++17", "-I", csrc, os.path.join(ROOT, "tools", "slice_qr_check.cpp"),
                    os.path.join(csrc, "slice_qr.cpp"), "-o", str(exe)], check=True, capture_output=True,
                   timeout=300)
    p = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
