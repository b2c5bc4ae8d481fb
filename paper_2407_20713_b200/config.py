"""Run configuration of the calibration front end: io::RunConfig and its JSON
loader (proj/include/sabr/io.hpp, proj/src/io.cpp:163-287), with the same
schema, defaults, unknown-key rejection and error messages, so a reference
config file drives this engine unchanged.  The B200-specific choices (device,
random stream, path-loop precision) are command-line flags, not config keys:
the reference's config contract (every unknown key is an error) stays intact.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field
from typing import Dict, Optional, Tuple

from .api import AnnealingSchedule, DomainError, SimulationPlan


class ConfigError(Exception):
    """io::config_error (io.hpp:26-29): CLI exit code 2."""


def _reject_unknown(obj: dict, known, where: str) -> None:  # io.cpp:163-170
    for key in obj:
        if key not in known:
            raise ConfigError(f"unknown key '{key}' in {where}")


def _as_int(v, where):
    if isinstance(v, bool) or not isinstance(v, (int, float)) or (isinstance(v, float) and not v.is_integer()):
        raise ConfigError(f"{where} must be an integer")
    return int(v)


def _as_float(v, where):
    if isinstance(v, bool) or not isinstance(v, (int, float)):
        raise ConfigError(f"{where} must be a number")
    return float(v)


_SCHEDULE_KEYS = {"t0": float, "cooling": float, "chain_length": int, "workers": int, "groups": int,
                  "t_min": float, "max_evals": int, "seed": int, "omp_threads": int}
_PLAN_KEYS = {"num_paths": int, "dt": float, "seed": int, "workers": int, "block_size": int}


def _parse_schedule(obj: dict) -> AnnealingSchedule:  # io.cpp:177-192
    _reject_unknown(obj, _SCHEDULE_KEYS, "annealing")
    s = AnnealingSchedule()
    for k, t in _SCHEDULE_KEYS.items():
        if k in obj:
            setattr(s, k, _as_int(obj[k], "annealing." + k) if t is int else _as_float(obj[k], "annealing." + k))
    return s


def _parse_plan(obj: dict, where: str) -> SimulationPlan:  # io.cpp:194-203
    _reject_unknown(obj, _PLAN_KEYS, where)
    p = SimulationPlan()
    for k, t in _PLAN_KEYS.items():
        if k in obj:
            setattr(p, k, _as_int(obj[k], f"{where}.{k}") if t is int else _as_float(obj[k], f"{where}.{k}"))
    return p


@dataclass
class RunConfig:
    """io::RunConfig (io.hpp:64-80), same defaults."""

    model: str = ""         # "static" | "case1" | "case2"
    technique: str = ""     # "T_I" | "T_II"
    surface_path: str = ""
    slice: int = 0
    fixed: Dict[str, float] = field(default_factory=dict)
    bounds: Dict[str, Tuple[float, float]] = field(default_factory=dict)
    schedule: AnnealingSchedule = field(default_factory=AnnealingSchedule)
    plan: SimulationPlan = field(default_factory=SimulationPlan)
    report_plan: Optional[SimulationPlan] = None
    output_dir: str = "."

    def validate(self) -> None:  # io.cpp:207-225
        if self.model not in ("static", "case1", "case2"):
            raise ConfigError("model must be one of static, case1, case2")
        if self.technique not in ("T_I", "T_II"):
            raise ConfigError("technique must be T_I or T_II")
        if self.technique == "T_II" and self.model != "case2":
            raise ConfigError("technique T_II is only wired up for the case2 model")
        for name, (lo, hi) in self.bounds.items():
            if not lo < hi:
                raise ConfigError(f"bounds for {name}: lower must be below upper")
        try:
            self.schedule.validate()
            self.plan.validate()
            if self.report_plan is not None:
                self.report_plan.validate()
        except DomainError as e:
            raise ConfigError(str(e)) from None


def parse_config_text(text: str) -> RunConfig:  # io.cpp:227-265
    try:
        obj = json.loads(text)
    except json.JSONDecodeError as e:
        raise ConfigError(f"config is not valid JSON: {e}") from None
    if not isinstance(obj, dict):
        raise ConfigError("config is not valid JSON: top level must be an object")
    _reject_unknown(obj, ("model", "technique", "surface", "slice", "fixed", "bounds", "annealing",
                          "simulation", "report_simulation", "output_dir"), "config")
    c = RunConfig()
    if "model" in obj:
        c.model = str(obj["model"])
    if "technique" in obj:
        c.technique = str(obj["technique"])
    if "surface" in obj:
        c.surface_path = str(obj["surface"])
    if "slice" in obj:
        c.slice = _as_int(obj["slice"], "slice")
    if "output_dir" in obj:
        c.output_dir = str(obj["output_dir"])
    for key, value in obj.get("fixed", {}).items():
        if isinstance(value, bool) or not isinstance(value, (int, float)):
            raise ConfigError(f"fixed.{key} must be a number")
        c.fixed[key] = float(value)
    for key, value in obj.get("bounds", {}).items():
        if not isinstance(value, list) or len(value) != 2:
            raise ConfigError(f"bounds.{key} must be [lower, upper]")
        c.bounds[key] = (_as_float(value[0], f"bounds.{key}"), _as_float(value[1], f"bounds.{key}"))
    if "annealing" in obj:
        c.schedule = _parse_schedule(obj["annealing"])
    if "simulation" in obj:
        c.plan = _parse_plan(obj["simulation"], "simulation")
    if "report_simulation" in obj:
        c.report_plan = _parse_plan(obj["report_simulation"], "report_simulation")
    c.validate()
    return c


def load_config(path: str) -> RunConfig:  # io.cpp:267-272
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise ConfigError(f"cannot open config {path}") from None
    return parse_config_text(text)


def apply_worker_env(c: RunConfig) -> Optional[int]:  # io.cpp:274-287
    env = os.environ.get("SABR_WORKERS")
    if env is None:
        return None
    if not env.isdigit() or int(env) < 1:
        raise ConfigError("SABR_WORKERS must be a positive integer")
    budget = int(env)
    # a thread budget on the CPU; the device engine's decomposition never depends on it
    c.schedule.omp_threads = budget
    c.plan.workers = budget
    if c.report_plan is not None:
        c.report_plan.workers = budget
    return budget
