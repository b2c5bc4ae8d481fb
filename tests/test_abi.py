"""The C-ABI boundary on a CPU-only host: the library loads, exports exactly
what include/sabr_b200.h declares, the ctypes mirror matches the C layouts,
host-only entry points behave like the reference, and compute entry points
fail loudly (no CPU fallback) when there is no GPU."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

import paper_2407_20713_b200 as pkg
from paper_2407_20713_b200 import _abi as A

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sabr_b200.h")


def declared_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"SABR_API\s+[\w\s\*]+?\b(sabr_\w+)\s*\(", text)))


def test_header_declares_exactly_the_exports():
    assert declared_functions() == sorted(A.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = A.load_library()
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", A.LIB_PATH], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert exported == set(declared_functions())  # nothing else leaks (hidden visibility)


def test_version():
    assert b"sm_100a" in A.load_library().sabr_version()


STRUCTS = ["sabr_surface", "sabr_schedule", "sabr_plan", "sabr_bounds", "sabr_fixed", "sabr_report_row",
           "sabr_report", "sabr_anneal_result", "sabr_timing", "sabr_level_record", "sabr_sa_state"]


def test_ctypes_mirror_matches_c_layout():
    src = '#include <stdio.h>\n#include <stddef.h>\n#include "sabr_b200.h"\nint main(void){\n'
    for s in STRUCTS:
        src += f'printf("{s} %zu\\n", sizeof({s}));\n'
        for f, _ in getattr(A, s)._fields_:
            src += f'printf("{s}.{f} %zu\\n", offsetof({s}, {f}));\n'
    src += "return 0;}\n"
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "layout.c")
        exe = os.path.join(d, "layout")
        open(c, "w").write(src)
        gcc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
        subprocess.run([gcc, "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
        lines = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    got = dict(zip(lines[0::2], (int(v) for v in lines[1::2])))
    for s in STRUCTS:
        cls = getattr(A, s)
        assert got[s] == C.sizeof(cls), s
        for f, _ in cls._fields_:
            assert got[f"{s}.{f}"] == getattr(cls, f).offset, f"{s}.{f}"


def test_black_scholes_host_entry_point():
    # black_scholes.cpp:20-35 / test_calibration.cpp:84-97
    s = pkg.parse_surface(os.path.join(ROOT, "tests", "data", "eurostoxx50.csv"))
    sl = s.slices[0]
    p = pkg.black_scholes_call(s.spot, sl.quotes[10].strike, sl.rate, sl.dividend, sl.maturity, sl.quotes[10].vol)
    assert abs(p - 134.605) <= 2e-5 * 134.605
    with pytest.raises(pkg.DomainError):
        pkg.black_scholes_call(-1.0, 100.0, 0.0, 0.0, 1.0, 0.2)


def test_surface_parse_errors_carry_line_numbers(tmp_path):
    # io::parse_surface_text grammar errors (io.cpp:68-119)
    bad = tmp_path / "bad.csv"
    bad.write_text("spot,100\nstrikes,absolute\nslice,1.0,1.0\n")
    with pytest.raises(pkg.NumericalError, match="line 3"):
        pkg.parse_surface(str(bad))
    bad.write_text("spot,100\nstrikes,percent\nslice,1.0,1.0,0.5\n90,20\n80,21\n")
    with pytest.raises(pkg.NumericalError, match="strictly increasing"):
        pkg.parse_surface(str(bad))
    bad.write_text("spot,100\nslice,1.0,1.0,0.5\n90,20\n")
    with pytest.raises(pkg.NumericalError, match="missing strikes header"):
        pkg.parse_surface(str(bad))


def _record(end_v, end_c, best_v, best_c, evals, dim=2, fill=0.0):
    r = A.sabr_level_record()
    r.end_value, r.end_chain, r.best_value, r.best_chain, r.evals = end_v, end_c, best_v, best_c, evals
    for i in range(dim):
        r.end_point[i] = fill + i
        r.best_point[i] = fill + 10 + i
    return r


def test_merge_rule_strict_less_lowest_chain_wins():
    """annealer.cpp:141-159: incumbent replaced only on strict '<'; among
    equal values the lowest chain index wins; evals add up; cap follows."""
    lib = A.load_library()
    st = A.sabr_sa_state()
    st.incumbent_value = 5.0
    st.best_value = 4.0
    st.evals = 1
    recs = (A.sabr_level_record * 3)(_record(3.0, 7, 2.0, 8, 100, fill=1.0),
                                     _record(3.0, 2, 2.0, 9, 100, fill=2.0),   # same value, lower chain
                                     _record(6.0, 40, 1.5, 41, 100, fill=3.0))
    tf = C.c_double()
    assert lib.sabr_merge_level_records(C.byref(st), recs, 3, 48, 10_000, 50, C.byref(tf)) == 0
    assert st.incumbent_value == 3.0 and st.incumbent[0] == 2.0  # chain 2 (rank 1) won the tie
    assert st.best_value == 1.5 and st.best[0] == 13.0
    assert st.evals == 301 and tf.value == 3.0 and st.levels_run == 1
    assert st.eval_cap == (10_000 - 301 + 47) // 48 and st.done == 0
    # not strictly better -> incumbent kept
    recs2 = (A.sabr_level_record * 1)(_record(3.0, 0, 9.0, 0, 10))
    lib.sabr_merge_level_records(C.byref(st), recs2, 1, 48, 10_000, 50, C.byref(tf))
    assert st.incumbent[0] == 2.0
    # budget exhausted -> done
    recs3 = (A.sabr_level_record * 1)(_record(9.0, 0, 9.0, 0, 10_000))
    lib.sabr_merge_level_records(C.byref(st), recs3, 1, 48, 10_000, 50, C.byref(tf))
    assert st.done == 1


@pytest.mark.skipif(os.environ.get("CUDA_VISIBLE_DEVICES", "x") != "" and os.path.exists("/dev/nvidia0"),
                    reason="a GPU is present")
def test_no_gpu_fails_loudly():
    with pytest.raises(pkg.api.CudaError):
        pkg.Engine(0)
