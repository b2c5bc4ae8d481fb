"""Generate tests/golden/*.json from the UNMODIFIED reference (oracle/_ref,
compiled from /root/reference/proj/src by oracle/Makefile).

  python tests/golden/make_golden.py

Doubles are stored as float.hex() strings so the fixtures round-trip exactly.
These fixtures pin the oracle restatement (tests/test_oracle.py) and travel
with the repo to hosts where /root/reference does not exist.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import paper_2407_20713_b200 as pkg  # noqa: E402
from paper_2407_20713_b200 import _abi as A  # noqa: E402
from oracles import DATA_DIR, Ref, atm_vol_guess, ref_parse_surface  # noqa: E402


def hx(a):
    if isinstance(a, (list, tuple, np.ndarray)):
        return [hx(v) for v in a]
    return float(a).hex()


def static_vectors(n, seed):
    rng = np.random.default_rng(seed)
    return np.column_stack([rng.uniform(1e-4, 2, n), rng.uniform(0, 1, n), rng.uniform(1e-4, 10, n),
                            rng.uniform(-1, 1, n)])


def case1_vectors(n, seed):
    rng = np.random.default_rng(seed)
    P = np.column_stack([rng.uniform(1e-4, 2, n), rng.uniform(0, 1, n), rng.uniform(-1, 1, n),
                         rng.uniform(1e-4, 10, n), rng.uniform(0, 150, n), rng.uniform(0, 150, n)])
    P[: n // 4, 4:] = rng.uniform(0, 0.1, (n // 4, 2))
    return P


def case2_vectors(n, seed):
    rng = np.random.default_rng(seed)
    lo = np.array([1e-4, 0, -1, -15, -1, 1e-4, -15, -1, 0, 0])
    hi = np.array([2, 1, 1, 15, 1, 10, 15, 1, 150, 150])
    P = lo + (hi - lo) * rng.random((n, 10))
    P[: n // 2, 3] *= 0.05
    P[: n // 2, 6] *= 0.05
    P[: n // 2, 8:] *= 0.02
    return np.column_stack([P, np.full(n, 2.0)])


def main():
    ref = Ref()
    eq = ref_parse_surface(os.path.join(DATA_DIR, "eurostoxx50.csv"))
    fx = ref_parse_surface(os.path.join(DATA_DIR, "eurusd.csv"))
    out = {"generator": "tests/golden/make_golden.py (oracle/_ref = unmodified reference)"}

    # surfaces as parsed by io::parse_surface (proj/src/io.cpp)
    out["surfaces"] = {name: {"spot": hx(s.spot),
                              "slices": [[hx(sl.maturity), hx(sl.rate), hx(sl.dividend),
                                          [[hx(q.strike), hx(q.vol)] for q in sl.quotes]] for sl in s.slices]}
                       for name, s in (("eurostoxx50", eq), ("eurusd", fx))}

    # cost functions (calibration.cpp:253-275 with :300-306 / :339-349)
    P4 = static_vectors(200, 42)
    P6 = case1_vectors(200, 43)
    out["cost_static"] = {"params": hx(P4), "eurostoxx50": [hx(ref.cost_static(eq, sl, P4)) for sl in range(4)],
                          "eurusd": [hx(ref.cost_static(fx, sl, P4)) for sl in range(4)]}
    out["cost_case1"] = {"params": hx(P6), "eurostoxx50": hx(ref.cost_case1(eq, P6)),
                         "eurusd": hx(ref.cost_case1(fx, P6))}
    # Case II feasibility (analytics.cpp:145-175)
    P11 = case2_vectors(400, 44)
    out["case2_feasible"] = {"params": hx(P11), "feasible": [bool(b) for b in ref.case2_feasible(P11)]}

    # RNG streams (rng.hpp)
    out["xoshiro"] = {f"{seed}_{stream}": hx(ref.xoshiro_uniforms(seed, stream, 8))
                      for seed, stream in ((0, 0), (1, 2), (42, 1 << 20), (2 ** 63 + 5, 12345))}

    # annealer on the closed forms of test_annealer.cpp (annealer.cpp:76-167)
    quick = dict(t0=5.0, cooling=0.9, chain_length=40, workers=8, t_min=1e-6, seed=1)
    cases = [("bowl3", A.OBJ_BOWL3, [-5] * 3, [5] * 3, [0, 0, 0], 0, {}),
             ("sinquad2_g3", A.OBJ_SINQUAD2, [-5, -5], [5, 5], [0, 0], 0, {"groups": 3, "seed": 7}),
             ("corner2_pred", A.OBJ_CORNER2, [-2, -2], [2, 2], [0, 0], A.PRED_SUM_LE_1, {}),
             ("nanright1", A.OBJ_NANRIGHT1, [-2], [2], [0], 0, {}),
             ("square1_budget", A.OBJ_SQUARE1, [-1], [1], [0.5], 0, {"max_evals": 500})]
    out["anneal_builtin"] = {}
    for name, obj, lo, hi, st, pred, kw in cases:
        s = pkg.AnnealingSchedule(**{**quick, **kw})
        r = ref.minimize_builtin(obj, lo, hi, s, st, predicate=pred)
        out["anneal_builtin"][name] = {
            "objective": obj, "lower": lo, "upper": hi, "start": st, "predicate": pred,
            "schedule": {**quick, **kw}, "best_point": hx(r.best_point), "best_value": hx(r.best_value),
            "evals": r.evals, "trace": [[hx(t), hx(f)] for t, f in r.temperature_trace]}

    # static T_I trajectory, C1 schedule (acceptance.cpp:318-323), equity slice 0
    out["anneal_static_c1"] = {}
    for seed in (1, 2, 3):
        s = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=32, t_min=1e-7, seed=seed)
        start = [atm_vol_guess(eq, 0), 1.0, 0.5, -0.3]
        r = ref.minimize_cost(A.MODEL_STATIC, eq, 0, [1e-4, 0, 1e-4, -1], [2, 1, 10, 1], s, start)
        out["anneal_static_c1"][str(seed)] = {
            "start": hx(start), "best_point": hx(r.best_point), "best_value": hx(r.best_value),
            "evals": r.evals, "trace_f": hx([f for _, f in r.temperature_trace])}

    # Monte Carlo streams (mc.cpp): terminal forwards and prices
    K_STATIC = pkg.StaticSabrParams(0.375162, 0.999999, 0.331441, -0.999999)
    K_CASE1 = pkg.CaseIParams(0.393329, 1.0, -1.0, 0.941565, 0.001, 1.246906)
    K_CASE2 = pkg.CaseIIParams(0.398436, 0.999579, -0.964678, 0.0, 0.101632, 1.285129, 1.302296,
                               -0.086294, 0.0, 2.059560, 0.495890)
    out["mc"] = {}
    for name, p in (("static", K_STATIC), ("case1", K_CASE1), ("case2", K_CASE2)):
        plan = pkg.SimulationPlan(num_paths=5000, seed=3, block_size=1000)
        t = ref.simulate_terminals(p, 2257.37, p.alpha, 0.495890, plan, serial=True)
        est = ref.price_european_batch(p, 2257.37, [2000.0, 2257.37, 2500.0], 0.018196, 0.034516, 0.495890, plan)
        out["mc"][name] = {"params": p.vector(), "plan": {"num_paths": 5000, "seed": 3, "block_size": 1000},
                           "terminals_head": hx(t[:64]), "terminals_tail": hx(t[-64:]),
                           "terminals_sum": hx(float(np.sum(t))),
                           "prices": [[hx(e.value), hx(e.std_error)] for e in est]}

    # price_cliquet (mc.cpp:275-320), the acceptance c9 spec
    K_FX1 = pkg.CaseIParams(0.155464, 0.971908, -0.642617, 0.800275, 0.001, 2.6093)
    out["cliquet"] = {}
    for name, dt in (("dt250", 1 / 250), ("dt007", 0.07)):
        plan = pkg.SimulationPlan(num_paths=3000, seed=3, block_size=1000, dt=dt)
        e = ref.price_cliquet(K_FX1, 1.2939, 0.010832, 0.006907, -0.02, 0.02, 0.0, 0.2, [0.25, 0.5, 0.75, 1.0],
                              plan)
        out["cliquet"][name] = {"dt": dt, "value": hx(e.value), "std_error": hx(e.std_error)}

    # Case II coefficient functionals and the calibrate_case2_formula objective
    P2 = np.array([[0.296790, 1.0, -0.360610, 15.0, -0.715716, 0.000100, -8.969205, 0.847244, 15.0, 15.0, 2.0],
                   [0.154037, 1.0, -0.693682, 0.345973, -0.200342, 7.541424, -0.992551, 0.339807, 0.0, 150.0,
                    2.0]])
    from oracles import ref_cost_case2_formula
    out["case2_formula"] = {"params": hx(P2),
                            "coeffs": [[hx(ref.dyn_coeffs_case2(p, T, 8)) for T in (0.25, 1.0, 2.0)] for p in P2],
                            "eurusd": hx(ref_cost_case2_formula(ref, fx, P2)),
                            "eurostoxx50": hx(ref_cost_case2_formula(ref, eq, P2))}

    # calibrate_* reports
    s = pkg.AnnealingSchedule(t0=1.0, cooling=0.8, chain_length=10, workers=4, t_min=1e-2, seed=1)
    rep = ref.calibrate_static_T1(fx, 0, {"nu": (0.01, 3.0)}, s, {"beta": 0.75, "rho": -0.4})
    out["calibrate_static_T1"] = {"params": {k: hx(v) for k, v in rep.params.items()},
                                  "final_cost": hx(rep.final_cost), "evals": rep.evals,
                                  "rows_model": hx([r.model for r in rep.rows])}
    surf = pkg.VolSurface(eq.spot, [eq.slices[2]])
    fixed = {"a": 0.0, "b": 0.0, "q_rho": 0.0, "q_nu": 0.0, "d_rho": 0.0, "d_nu": 0.0, "beta": 1.0}
    s2 = pkg.AnnealingSchedule(t0=2.0, cooling=0.5, chain_length=4, workers=6, t_min=0.2, seed=3)
    plan = pkg.SimulationPlan(num_paths=2048, seed=1)
    rep = ref.calibrate_case2_T2(surf, None, s2, plan, fixed)
    out["calibrate_case2_T2"] = {"params": {k: hx(v) for k, v in rep.params.items()},
                                 "final_cost": hx(rep.final_cost), "evals": rep.evals,
                                 "rows_model": hx([r.model for r in rep.rows])}

    path = os.path.join(HERE, "golden.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
