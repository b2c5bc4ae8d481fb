"""Accuracy of the MC kernels' table log and Goldschmidt sqrt
(device_common.cuh log_tab / sqrt_pos, Box-Muller's radius, mc.cpp:30-36):
their host builds against x86 long double over u1 = 1 - k 2^-53 in every
binade (tools/mathtab_check.cpp): < 1 ulp, sqrt(0) = 0."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not available")
def test_log_tab_and_sqrt_pos_accuracy(tmp_path):
    exe = tmp_path / "mathtab_check"
    subprocess.run(["nvcc", "-x", "cu", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"), "-I",
                    os.path.join(ROOT, "paper_2407_20713_b200", "csrc"), os.path.join(ROOT, "tools", "mathtab_check.cpp"),
                    "-o", str(exe)], check=True, capture_output=True, timeout=300)
    p = subprocess.run([str(exe), "3000000"], capture_output=True, text=True, timeout=300)
    print(p.stdout)
    assert p.returncode == 0, p.stdout + p.stderr
