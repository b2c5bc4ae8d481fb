"""Run-config loader and command-line front end (config.py, cli.py) against the
reference's io / sabr_cli contract (proj/tests/test_io.cpp:112-229,
proj/src/io.cpp:163-357, proj/tools/sabr_cli.cpp)."""
import json
import os
import subprocess
import sys

import pytest

import paper_2407_20713_b200 as pkg
from paper_2407_20713_b200 import cli
from paper_2407_20713_b200.config import ConfigError, parse_config_text

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DATA = os.path.join(ROOT, "tests", "data")


def run_cli(args, expected_exit, cwd=ROOT):
    p = subprocess.run([sys.executable, "-m", "paper_2407_20713_b200", *args], cwd=cwd, capture_output=True,
                       text=True, timeout=600)
    assert p.returncode == expected_exit, (p.returncode, p.stdout[-2000:], p.stderr[-2000:])
    return p.stdout + p.stderr


def test_config_rejects_unknown_keys_at_every_level():  # test_io.cpp:112-140
    cfg = parse_config_text('''{
        "model": "static", "technique": "T_I", "surface": "s.csv", "slice": 1,
        "fixed": {"beta": 1.0},
        "bounds": {"nu": [0.01, 5.0]},
        "annealing": {"t0": 2.0, "cooling": 0.96, "chain_length": 50, "workers": 8, "seed": 3}}''')
    assert cfg.model == "static" and cfg.slice == 1 and cfg.fixed["beta"] == 1.0
    assert cfg.bounds["nu"][0] == 0.01 and cfg.schedule.t0 == 2.0 and cfg.schedule.seed == 3
    for bad, msg in (('{"model": "static", "typo": 1}', "unknown key 'typo' in config"),
                     ('{"model": "static", "surface": "s", "annealing": {"warmth": 2}}',
                      "unknown key 'warmth' in annealing"),
                     ('{"model": "static", "surface": "s", "simulation": {"paths": 1}}',
                      "unknown key 'paths' in simulation"),
                     ("{not json", "config is not valid JSON")):
        with pytest.raises(ConfigError, match=msg):
            parse_config_text(bad)


def test_config_validation():  # test_io.cpp:142-160
    base = '{"model": "%s", "technique": "%s", "surface": "s.csv"}'
    parse_config_text(base % ("static", "T_I")).validate()
    with pytest.raises(ConfigError, match="model must be one of"):
        parse_config_text(base % ("pricer", "T_I"))
    with pytest.raises(ConfigError, match="only wired up for the case2 model"):
        parse_config_text(base % ("static", "T_II"))
    parse_config_text(base % ("case2", "T_II")).validate()
    with pytest.raises(ConfigError, match="bounds for nu: lower must be below upper"):
        parse_config_text('{"model": "static", "technique": "T_I", "surface": "s", "bounds": {"nu": [5.0, 0.01]}}')
    with pytest.raises(ConfigError, match="cooling"):  # AnnealingSchedule::validate -> config_error
        parse_config_text('{"model": "static", "technique": "T_I", "annealing": {"cooling": 1.5}}')


def test_report_serialization():  # test_io.cpp:162-185
    rep = pkg.CalibrationReport(model="static", technique="T_I", quantity="vol",
                                params={"alpha": 0.3, "beta": 1.0}, final_cost=1.5e-3,
                                rows=[pkg.ReportRow(0.25, 90.0, 0.21, 0.209, -0.0047619047619),
                                      pkg.ReportRow(0.25, 100.0, 0.20, 0.201, 0.005)],
                                mean_rel_error=4.88e-3, max_rel_error=5.0e-3, wall_seconds=1.25, evals=1234, seed=7)
    csv = cli.report_to_csv(rep)
    assert "maturity,strike,market,model,rel_error" in csv and "\n0.25,90,0.21,0.209,-0.0047619047619\n" in csv
    assert "# param,alpha,0.3\n" in csv and "# evals,1234\n" in csv
    obj = json.loads(cli.report_to_json(rep))
    assert obj["schema_version"] == 1 and obj["params"]["alpha"] == 0.3 and len(obj["rows"]) == 2


def test_cli_exit_codes(tmp_path):  # test_io.cpp:187-205
    run_cli(["calibrate", "--config", "/nonexistent.json"], cli.EXIT_CONFIG)
    bad = tmp_path / "bad.csv"
    bad.write_text("spot,100\nstrikes,percent\nslice,1.0,1.0,0.0\n90,notanumber\n")
    cfg = tmp_path / "cfg.json"
    cfg.write_text(json.dumps({"model": "static", "technique": "T_I", "surface": str(bad),
                               "fixed": {"alpha": 0.3, "beta": 1.0, "nu": 0.5, "rho": -0.5}}))
    assert "line 4" in run_cli(["calibrate", "--config", str(cfg)], cli.EXIT_PARSE)
    run_cli(["calibrate"], cli.EXIT_CONFIG)  # --config is required
    cfg.write_text(json.dumps({"model": "static", "technique": "T_I", "surface": str(bad), "fixed": {"beta": 1.0}}))
    assert "eval mode: parameter 'alpha' is not fixed" in run_cli(["eval", "--config", str(cfg)], cli.EXIT_CONFIG)
    assert "--fixed expects name=value" in run_cli(["calibrate", "--config", str(cfg), "--fixed", "beta"],
                                                   cli.EXIT_CONFIG)


@pytest.mark.gpu
def test_cli_smile_on_fixed_parameters(tmp_path, ref):  # test_io.cpp:207-229
    params = tmp_path / "p.json"
    params.write_text(json.dumps({"model": "static", "params": {"alpha": 0.146859, "beta": 1.0, "nu": 0.911966,
                                                                "rho": -0.447718}}))
    out = run_cli(["smile", "--params", str(params), "--surface", os.path.join(DATA, "eurusd.csv")], cli.EXIT_OK)
    lines = out.strip().splitlines()
    assert lines[0] == "maturity,strike,vol" and len(lines) >= 20
    fx = pkg.parse_surface(os.path.join(DATA, "eurusd.csv"))
    rows = [tuple(float(x) for x in ln.split(",")) for ln in lines[1:]]
    assert len(rows) == fx.total_quotes()
    T, K, v = rows[0]
    want = ref.static_vol([0.146859, 1.0, 0.911966, -0.447718], fx.slices[0].quotes[0].strike, fx.forward(0),
                          fx.slices[0].maturity)
    assert abs(v - want) <= 5e-6 * want  # %g output: 6 significant digits


@pytest.mark.gpu
def test_cli_calibrate_writes_reference_reports(tmp_path):
    cfg = tmp_path / "run.json"
    cfg.write_text(json.dumps({"model": "static", "technique": "T_I", "surface": os.path.join(DATA, "eurusd.csv"),
                               "slice": 2, "annealing": {"t0": 2.0, "cooling": 0.8, "chain_length": 20,
                                                         "workers": 64, "t_min": 1e-3, "seed": 5},
                               "output_dir": str(tmp_path)}))
    out = run_cli(["calibrate", "--config", str(cfg)], cli.EXIT_OK)
    assert "static / T_I on 19 quotes" in out
    rep = json.loads((tmp_path / "report_static_T_I.json").read_text())
    eng = pkg.Engine(0)
    fx = pkg.parse_surface(os.path.join(DATA, "eurusd.csv"))
    direct = eng.calibrate_static_T1(fx, 2, None, pkg.AnnealingSchedule(t0=2.0, cooling=0.8, chain_length=20,
                                                                         workers=64, t_min=1e-3, seed=5), None)
    eng.close()
    assert rep["final_cost"] == direct.final_cost and rep["evals"] == direct.evals
    assert (tmp_path / "report_static_T_I.csv").read_text().startswith("# model,static\n")
