"""Command-line front end: calibrate, eval, price, smile (proj/tools/sabr_cli.cpp)
over the B200 engine.

  python -m paper_2407_20713_b200 calibrate --config run.json [--seed S] [--workers W]
                                            [--output DIR] [--fixed beta=1 ...]
  python -m paper_2407_20713_b200 eval      --config run.json ...
  python -m paper_2407_20713_b200 price     --params p.json --contract c.json [--config run.json]
  python -m paper_2407_20713_b200 smile     --params p.json --surface s.csv [--grid N] [--out F]

The reference's config files, parameter files, contract files, report files
(report_<model>_<technique>.{csv,json}) and exit codes (0 ok, 2 config error,
3 parse error, 4 any other error; sabr_cli.cpp:303-317, io.hpp:34-39) are kept.
B200 choices are flags, so the config contract (unknown keys rejected) stays:
--device N, --rng {xoshiro,philox}, --precision {fp64,fp32}.
"""
from __future__ import annotations

import argparse
import json
import math
import sys
import time
from typing import List, Optional

import numpy as np

from . import _abi as A
from .api import (CalibrationReport, CaseIIParams, CaseIParams, Engine, ParseError, PriceEstimate,
                  StaticSabrParams, VolQuote, VolSlice, VolSurface, parse_surface)
from .config import ConfigError, RunConfig, apply_worker_env, load_config

EXIT_OK, EXIT_CONFIG, EXIT_PARSE, EXIT_NUMERICAL = 0, 2, 3, 4

PARAM_NAMES = {
    "static": ["alpha", "beta", "nu", "rho"],
    "case1": ["alpha", "beta", "rho0", "nu0", "a", "b"],
    "case2": ["alpha", "beta", "rho0", "q_rho", "d_rho", "nu0", "q_nu", "d_nu", "a", "b"],
}


def fmt(x: float) -> str:
    """io.cpp:17-21 (std::to_chars shortest round trip) == Python repr."""
    if x != x:
        return "nan"
    if math.isinf(x):
        return "inf" if x > 0 else "-inf"
    r = repr(float(x))
    return r[:-2] if r.endswith(".0") else r


# ---------------------------------------------------------------- reports ---
def report_to_csv(rep: CalibrationReport) -> str:  # io.cpp:289-307
    out = [f"# model,{rep.model}", f"# technique,{rep.technique}", f"# quantity,{rep.quantity}"]
    out += [f"# param,{k},{fmt(v)}" for k, v in sorted(rep.params.items())]
    out += [f"# final_cost,{fmt(rep.final_cost)}", f"# mean_rel_error,{fmt(rep.mean_rel_error)}",
            f"# max_rel_error,{fmt(rep.max_rel_error)}", f"# evals,{rep.evals}", f"# seed,{rep.seed}",
            "maturity,strike,market,model,rel_error"]
    out += [f"{fmt(r.maturity)},{fmt(r.strike)},{fmt(r.market)},{fmt(r.model)},{fmt(r.rel_error)}"
            for r in rep.rows]
    return "\n".join(out) + "\n"


def report_to_json(rep: CalibrationReport) -> str:  # io.cpp:309-331 (nlohmann dump(2): sorted keys)
    obj = {"schema_version": 1, "model": rep.model, "technique": rep.technique, "quantity": rep.quantity,
           "params": dict(sorted(rep.params.items())), "final_cost": rep.final_cost,
           "mean_rel_error": rep.mean_rel_error, "max_rel_error": rep.max_rel_error,
           "wall_seconds": rep.wall_seconds, "evals": rep.evals, "seed": rep.seed,
           "rows": [{"maturity": r.maturity, "strike": r.strike, "market": r.market, "model": r.model,
                     "rel_error": r.rel_error} for r in rep.rows]}
    return json.dumps(obj, indent=2, sort_keys=True) + "\n"


def write_report(rep: CalibrationReport, stem: str) -> None:  # io.cpp:333-342
    for ext, text in ((".csv", report_to_csv(rep)), (".json", report_to_json(rep))):
        try:
            with open(stem + ext, "w") as f:
                f.write(text)
        except OSError:
            raise RuntimeError(f"cannot write {stem}{ext}") from None


def price_to_json(est: PriceEstimate, label: str, seed: int, dt: float, wall: float) -> str:  # io.cpp:344-357
    obj = {"schema_version": 1, "label": label, "value": est.value, "std_error": est.std_error,
           "num_paths": est.num_paths, "dt": dt, "seed": seed, "wall_seconds": wall}
    return json.dumps(obj, indent=2, sort_keys=True) + "\n"


# -------------------------------------------------------------- commands ---
def load_with_overrides(args) -> RunConfig:  # sabr_cli.cpp:38-64
    c = load_config(args.config)
    apply_worker_env(c)
    if args.seed is not None:
        c.schedule.seed = args.seed
        c.plan.seed = args.seed
        if c.report_plan is not None:
            c.report_plan.seed = args.seed
    if args.workers is not None:
        c.schedule.omp_threads = args.workers
        c.plan.workers = args.workers
        if c.report_plan is not None:
            c.report_plan.workers = args.workers
    if args.output is not None:
        c.output_dir = args.output
    for kv in args.fixed or []:
        eq = kv.find("=")
        if eq <= 0:
            raise ConfigError(f"--fixed expects name=value, got '{kv}'")
        try:
            c.fixed[kv[:eq]] = float(kv[eq + 1:])
        except ValueError:
            raise ConfigError(f"--fixed value is not a number in '{kv}'") from None
    for plan in (c.plan, c.report_plan):
        if plan is not None:
            plan.rng = args.rng
            plan.precision = args.precision
    return c


class _LazyEngine:
    """The device context, created only once the inputs have been parsed (so
    config and parse errors never need a GPU)."""

    def __init__(self, device: int):
        self.device, self.eng = device, None

    def __call__(self) -> Engine:
        if self.eng is None:
            self.eng = Engine(self.device)
        return self.eng

    def close(self):
        if self.eng is not None:
            self.eng.close()


def run_calibration(engine: _LazyEngine, c: RunConfig) -> CalibrationReport:  # sabr_cli.cpp:66-80
    surface = parse_surface(c.surface_path)
    eng = engine()
    if c.model == "static":
        return eng.calibrate_static_T1(surface, c.slice, c.bounds, c.schedule, c.fixed)
    if c.model == "case1":
        return eng.calibrate_dynamic_case1_T1(surface, c.bounds, c.schedule, c.fixed)
    if c.technique == "T_I":
        return eng.calibrate_case2_formula(surface, c.bounds, c.schedule, c.fixed)
    return eng.calibrate_case2_T2(surface, c.bounds, c.schedule, c.plan, c.fixed, c.report_plan)


def print_summary(rep: CalibrationReport) -> None:  # sabr_cli.cpp:82-93
    print(f"{rep.model} / {rep.technique} on {len(rep.rows)} quotes")
    for name, value in sorted(rep.params.items()):
        print(f"  {name} = {value:.6g}")
    print(f"  final_cost     = {rep.final_cost:.6g}\n  mean_rel_error = {rep.mean_rel_error:.6g}\n"
          f"  max_rel_error  = {rep.max_rel_error:.6g}\n  evals          = {rep.evals}\n"
          f"  wall_seconds   = {rep.wall_seconds:.6g}")


def cmd_calibrate(eng: _LazyEngine, args, eval_only: bool) -> int:  # sabr_cli.cpp:143-164
    c = load_with_overrides(args)
    if eval_only:
        for name in PARAM_NAMES[c.model]:
            if name not in c.fixed:
                raise ConfigError(f"eval mode: parameter '{name}' is not fixed")
    rep = run_calibration(eng, c)
    print_summary(rep)
    write_report(rep, f"{c.output_dir}/report_{rep.model}_{rep.technique}")
    return EXIT_OK


def load_json_file(path: str):  # sabr_cli.cpp:95-103
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise ParseError(f"cannot open {path}") from None
    try:
        return json.loads(text)
    except json.JSONDecodeError as e:
        raise ParseError(f"{path}: {e}") from None


def need(obj: dict, key: str, where: str) -> float:  # sabr_cli.cpp:105-109
    if key not in obj:
        raise ConfigError(f"{where}: missing '{key}'")
    return float(obj[key])


def load_params(obj: dict, horizon: float):  # sabr_cli.cpp:111-141 (validation: the engine's)
    model = obj.get("model", "")
    if "params" not in obj:
        raise ConfigError("params file: missing 'params'")
    if model not in PARAM_NAMES:
        raise ConfigError("params file: model must be static, case1 or case2")
    v = [need(obj["params"], k, model) for k in PARAM_NAMES[model]]
    if model == "static":
        return model, StaticSabrParams(*v)
    if model == "case1":
        return model, CaseIParams(*v)
    return model, CaseIIParams(*v, horizon)


def cmd_price(engine: _LazyEngine, args) -> int:  # sabr_cli.cpp:166-204
    from .api import SimulationPlan

    if args.config:
        plan = load_with_overrides(args).plan
    else:
        plan = SimulationPlan(rng=args.rng, precision=args.precision)
        if args.seed is not None:
            plan.seed = args.seed
        if args.workers is not None:
            plan.workers = args.workers
    contract = load_json_file(args.contract)
    kind = contract.get("type", "")
    spot, rate, div = (need(contract, k, "contract") for k in ("spot", "rate", "dividend"))
    if kind == "european":
        horizon = need(contract, "maturity", "contract")
    elif kind == "cliquet":
        if "reset_dates" not in contract:
            raise ConfigError("contract: missing 'reset_dates'")
        horizon = float(contract["reset_dates"][-1])
    else:
        raise ConfigError("contract: type must be european or cliquet")
    _, params = load_params(load_json_file(args.params), horizon)
    eng = engine()
    t0 = time.perf_counter()
    if kind == "european":
        est = eng.price_european_call(params, spot, need(contract, "strike", "contract"), rate, div, horizon, plan)
    else:
        est = eng.price_cliquet(params, spot, rate, div, need(contract, "local_floor", "contract"),
                                need(contract, "local_cap", "contract"), need(contract, "global_floor", "contract"),
                                need(contract, "global_cap", "contract"),
                                [float(x) for x in contract["reset_dates"]], plan)
    sys.stdout.write(price_to_json(est, kind, plan.seed, plan.dt, time.perf_counter() - t0))
    return EXIT_OK


def cmd_smile(engine: _LazyEngine, args) -> int:  # sabr_cli.cpp:206-264
    surface = parse_surface(args.surface)
    horizon = surface.slices[-1].maturity
    model, params = load_params(load_json_file(args.params), horizon)
    eng = engine()
    # the evaluation grid as a surface (the vol column is a placeholder)
    grid = VolSurface(surface.spot)
    for sl in surface.slices:
        ks = [q.strike for q in sl.quotes]
        if args.grid > 0:
            lo, hi = ks[0], ks[-1]
            ks = [lo if args.grid == 1 else lo + (hi - lo) * j / (args.grid - 1) for j in range(args.grid)]
        grid.slices.append(VolSlice(sl.maturity, sl.rate, sl.dividend, [VolQuote(k, 1.0) for k in ks]))
    lines = ["maturity,strike,vol"]
    if model == "static":  # one slice per call (Eq. 7 on the slice's own forward)
        p = np.array([[params.alpha, params.beta, params.nu, params.rho]])
        for i, sl in enumerate(grid.slices):
            vols = eng.implied_vol_batch(A.MODEL_STATIC, grid, p, slice=i)[0]
            lines += [f"{sl.maturity:g},{q.strike:g},{v:g}" for q, v in zip(sl.quotes, vols)]
    else:
        kind = A.MODEL_CASE1 if model == "case1" else A.MODEL_CASE2
        vec = [getattr(params, k) for k in PARAM_NAMES[model]] + ([horizon] if model == "case2" else [])
        vols = eng.implied_vol_batch(kind, grid, np.array([vec]))[0]
        j = 0
        for sl in grid.slices:
            for q in sl.quotes:
                lines.append(f"{sl.maturity:g},{q.strike:g},{vols[j]:g}")
                j += 1
    text = "\n".join(lines) + "\n"
    if not args.out or args.out == "-":
        sys.stdout.write(text)
    else:
        try:
            with open(args.out, "w") as f:
                f.write(text)
        except OSError:
            raise RuntimeError(f"cannot write {args.out}") from None
    return EXIT_OK


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # CLI11 ParseError -> usage + kExitConfig (sabr_cli.cpp:294-299)
        self.print_usage(sys.stderr)
        sys.stderr.write(f"{self.prog}: error: {message}\n")
        raise SystemExit(EXIT_CONFIG)


def build_parser() -> argparse.ArgumentParser:
    ap = _Parser(prog="python -m paper_2407_20713_b200",
                 description="SABR volatility toolkit on B200: calibration and Monte Carlo pricing")
    sub = ap.add_subparsers(dest="cmd", required=True, parser_class=_Parser)

    def common(p, need_config=True):
        p.add_argument("--config", required=need_config, default=None, help="run configuration JSON")
        p.add_argument("--seed", type=int, default=None, help="override annealing and simulation seeds")
        p.add_argument("--workers", type=int, default=None, help="override the thread budget")
        p.add_argument("--output", default=None, help="report output directory")
        p.add_argument("--fixed", action="append", help="pin a parameter, e.g. --fixed beta=1 (repeatable)")

    def device(p):
        p.add_argument("--device", type=int, default=0, help="CUDA device ordinal")
        p.add_argument("--rng", choices=["xoshiro", "philox"], default="xoshiro",
                       help="MC stream: the reference's xoshiro blocks, or counter-based Philox")
        p.add_argument("--precision", choices=["fp64", "fp32"], default="fp64", help="MC path-loop arithmetic")

    for name, helptext in (("calibrate", "fit a model to a surface"),
                           ("eval", "tabulate model vs market (all params fixed)")):
        p = sub.add_parser(name, help=helptext)
        common(p)
        device(p)
    p = sub.add_parser("price", help="Monte Carlo price one contract")
    common(p, need_config=False)
    device(p)
    p.add_argument("--params", required=True, help="model parameter JSON")
    p.add_argument("--contract", required=True, help="contract JSON")
    p = sub.add_parser("smile", help="emit model implied vols on a grid")
    p.add_argument("--params", required=True, help="model parameter JSON")
    p.add_argument("--surface", required=True, help="surface CSV (maturities and strikes)")
    p.add_argument("--grid", type=int, default=0, help="dense strikes per maturity (0 = quotes)")
    p.add_argument("--out", default="-", help="output CSV path ('-' for stdout)")
    p.add_argument("--device", type=int, default=0, help="CUDA device ordinal")
    return ap


def main(argv: Optional[List[str]] = None) -> int:
    args = build_parser().parse_args(argv)
    eng = _LazyEngine(args.device)
    try:
        try:
            if args.cmd in ("calibrate", "eval"):
                return cmd_calibrate(eng, args, args.cmd == "eval")
            if args.cmd == "price":
                return cmd_price(eng, args)
            return cmd_smile(eng, args)
        finally:
            eng.close()
    except ConfigError as e:
        sys.stderr.write(f"config error: {e}\n")
        return EXIT_CONFIG
    except ParseError as e:
        sys.stderr.write(f"parse error: {e}\n")
        return EXIT_PARSE
    except Exception as e:  # std::exception
        sys.stderr.write(f"error: {e}\n")
        return EXIT_NUMERICAL
