"""The drop-in, end to end: the reference's own objects linked with
integration/sabr_b200_adapter.cpp (oracle/Makefile target ``adapter``).  The
binary calls sabr::calibrate_* (the reference, CPU) and sabr::b200::calibrate_*
(the adapter over include/sabr_b200.h, GPU) on the same surfaces, schedules and
seeds and prints both CalibrationReports; they must agree the way the engine
agrees with the reference everywhere else: the same trajectory (evals), the
same parameters and cost to rounding, and the reference's exception types for
its error cases (proj/tests/test_calibration.cpp:212-225).  The same for the
Monte Carlo operator (mc.hpp:66-84): prices, standard errors and terminals
on the reference's streams."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "adapter_check")


@pytest.fixture(scope="module")
def cases():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/adapter_check not built (needs /root/reference at build time)")
    out = subprocess.run([BIN, os.path.join(ROOT, "tests", "data")], capture_output=True, text=True,
                         timeout=900, check=True).stdout
    return {c["case"]: c for c in map(json.loads, out.splitlines())}


@pytest.mark.parametrize("name,cost_tol,param_tol", [("static_T1", 1e-12, 1e-9),
                                                     ("case1_T1", 1e-12, 1e-9),
                                                     ("case2_T2", 1e-10, 1e-9),
                                                     ("case2_formula", 1e-10, 1e-7),
                                                     ("evaluate_case1", 1e-12, 0.0),
                                                     ("evaluate_case2_prices", 1e-10, 0.0)])
def test_adapter_matches_reference(cases, name, cost_tol, param_tol):
    c = cases[name]
    ref, gpu = c["ref"], c["b200"]
    assert gpu["model"] == ref["model"]
    assert gpu["evals"] == ref["evals"]
    assert gpu["params"].keys() == ref["params"].keys()
    rc, gc = float.fromhex(ref["cost"]), float.fromhex(gpu["cost"])
    assert abs(gc - rc) <= cost_tol * max(1.0, abs(rc))
    for k in ref["params"]:
        r, g = float.fromhex(ref["params"][k]), float.fromhex(gpu["params"][k])
        assert abs(g - r) <= param_tol * max(1.0, abs(r)), k
    assert len(gpu["rows"]) == len(ref["rows"])
    for r, g in zip(ref["rows"], gpu["rows"]):
        r, g = float.fromhex(r), float.fromhex(g)
        assert abs(g - r) <= 1e-8 * max(1.0, abs(r))


@pytest.mark.parametrize("name", ["mc_static", "mc_case1", "mc_case2", "mc_cliquet"])
def test_adapter_mc_matches_reference(cases, name):
    """mc::price_european_batch / price_cliquet through the adapter: the
    reference's streams, prices and standard errors to 1e-11 relative."""
    c = cases[name]
    assert len(c["b200"]) == len(c["ref"])
    for (rv, rs), (gv, gs) in zip(c["ref"], c["b200"]):
        for r, g in ((rv, gv), (rs, gs)):
            r, g = float.fromhex(r), float.fromhex(g)
            assert abs(g - r) <= 1e-11 * max(abs(r), 1e-12), (name, r, g)


def test_adapter_mc_terminals(cases):
    c = cases["mc_terminals"]
    assert c["n"] == 10000
    assert c["max_rel"] <= 1e-12


def test_adapter_error_types(cases):
    c = cases["errors"]
    assert c["b200"] == c["ref"]
    assert c["ref"] == ["out_of_range", "domain_error", "domain_error", "domain_error"]
