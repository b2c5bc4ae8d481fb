"""The reference's own unit tests and CLI, compiled unchanged against the
drop-in dispatch (make -C oracle dropin), on the CPU backend (SABR_BACKEND
unset): the doctest and CLI11 shims of oracle/dropin/ reproduce the harness
the reference's CMake expects (proj/tests/CMakeLists.txt:1-16), so all 61
cases pass, including the CLI tests that run sabr_cli through popen
(test_io.cpp:187-229).  tests/test_gpu_reference_suites.py runs the same
binaries through the engine."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DROP = os.path.join(ROOT, "oracle", "_ref", "dropin")


def binary(name):
    path = os.path.join(DROP, name)
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (make -C oracle dropin needs /root/reference at build time)")
    return path


def cpu_env():
    env = dict(os.environ)
    env.pop("SABR_BACKEND", None)
    return env


def test_reference_unit_tests_pass_on_the_cpu_backend():
    p = subprocess.run([binary("unit_tests")], env=cpu_env(), capture_output=True, text=True, timeout=900)
    passed = [l for l in p.stdout.splitlines() if l.startswith("[doctest-shim] PASS ")]
    failed = [l for l in p.stdout.splitlines() if l.startswith("[doctest-shim] FAIL ")]
    assert p.returncode == 0 and len(passed) == 61 and not failed, p.stdout[-3000:]


@pytest.mark.parametrize("crit", [1, 2, 4, 5])
def test_reference_acceptance_criteria_on_the_cpu_backend(crit):
    """The deterministic formula criteria (acceptance.cpp:88-215)."""
    p = subprocess.run([binary("acceptance"), str(crit)], env=cpu_env(), capture_output=True, text=True,
                       timeout=600)
    assert f"criterion {crit}: PASS" in p.stdout, p.stdout[-2000:]


def test_reference_cli_through_the_cli11_shim(tmp_path):
    """sabr_cli's exit codes (sabr_cli.cpp:294-317, io.hpp kExit*) and an
    evaluation-mode report through the reference's own io::write_report."""
    cli = binary("sabr_cli")
    run = lambda *a: subprocess.run([cli, *a], env=cpu_env(), capture_output=True, text=True, timeout=300)
    assert run().returncode == 2                             # a subcommand is required
    assert run("calibrate").returncode == 2                  # --config is required
    assert run("calibrate", "--config", "/nonexistent.json").returncode == 2
    assert run("calibrate", "--bogus").returncode == 2
    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps({"model": "static", "technique": "T_I", "slice": 2, "output_dir": str(tmp_path),
                               "surface": os.path.join(ROOT, "tests", "data", "eurostoxx50.csv")}))
    p = run("eval", "--config", str(cfg), "--fixed", "alpha=0.289271", "--fixed", "beta=1", "--fixed",
            "nu=0.30856", "--fixed", "rho=-0.999729")
    assert p.returncode == 0, p.stdout + p.stderr
    csv = (tmp_path / "report_static_T_I.csv").read_text()
    assert "# evals,1\n" in csv and csv.count("\n") == 12 + 1 + 21  # 12 "#" lines, header, 21 quotes
    assert run("eval", "--config", str(cfg), "--fixed", "alpha=0.3").returncode == 2  # not all fixed
