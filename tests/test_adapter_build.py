"""The reference-side adapter (integration/sabr_b200_adapter.{hpp,cpp} and
its checker integration/adapter_check.cpp) compiles against the reference's
own headers and the C-ABI header - the drop-in a maintainer would add to
proj/src.  CPU only (g++ -fsyntax-only); skipped where the reference tree is
absent (the GPU box).  The GPU run is tests/test_gpu_adapter.py."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"


@pytest.mark.skipif(not os.path.isdir(REF_INC) or shutil.which("g++") is None,
                    reason="reference headers or g++ not available")
@pytest.mark.parametrize("src", ["sabr_b200_adapter.cpp", "adapter_check.cpp"])
def test_adapter_compiles_against_reference_headers(src):
    cmd = ["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Werror", "-I", REF_INC,
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(ROOT, "integration"),
           os.path.join(ROOT, "integration", src)]
    json_dir = next((d for d in ("/usr/include", "/usr/local/include")
                     if os.path.exists(os.path.join(d, "nlohmann", "json.hpp"))), None)
    if json_dir:
        cmd[4:4] = ["-I", json_dir]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-3000:]
