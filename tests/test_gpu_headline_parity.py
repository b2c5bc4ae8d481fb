"""The BASELINE.json configurations at their named shapes, against the compiled
reference (oracle/_ref) on the same inputs, seeds and schedules.

* C2 (static Hagan, EUR/USD, 1e5 chains = workers 12500 x groups 8): every
  slice with the C2 schedule capped at max_evals = 2e7 + 1 (the first two
  temperature levels: 1042 CTAs, the last-CTA merge, the per-level eval cap of
  annealer.cpp:102-105 and the group-ordered reduction of annealer.cpp:141-152
  all at full width), and one slice for the whole 412-level run (slow).
* C3 (Case I, EUR/USD) with beta free (calibration.cpp:325-365): the
  acceptance schedule (32 chains, 1e6 evals) and the 1e5-chain shape capped at
  one level.
* C5 (full Case II T_II, 20x30 surface): one SA step of 125,000 chains (the
  per-GPU share of 1e6 chains on 8 GPUs).  In the default Case II box the
  reference aborts (its mc runtime_error escapes the OpenMP region); the
  engine reports the same error as NumericalError.  The parity run uses the
  bench's box (+-2% of the default widths around the published FX fit).

Decisions (evals, trace length) must be identical; values agree to the
factored-cost tolerance (the slice cost differs from the
reference's per-quote sum by <= ~1e-14 relative)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2407_20713_b200 as pkg

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DATA = os.path.join(ROOT, "tests", "data")


def assert_same_anneal(g, r, cost_rtol=1e-12, param_atol=1e-9, trace_rtol=1e-12):
    """g: the engine's calibrate report (trace on); r: the reference annealer's
    result on the reference objective (same run as its calibrate_*)."""
    assert g.evals == r.evals
    assert len(g.temperature_trace) == len(r.temperature_trace)
    for (tg, fg), (tr, fr) in zip(g.temperature_trace, r.temperature_trace):
        assert tg == tr  # the schedule: repeated multiplication (annealer.cpp:99-100)
        assert abs(fg - fr) <= trace_rtol * max(abs(fr), 1e-12), (tg, fg, fr)
    assert abs(g.final_cost - r.best_value) <= cost_rtol * abs(r.best_value), (g.final_cost, r.best_value)
    gp = [g.params[k] for k in ("alpha", "beta", "nu", "rho")]
    for a, b in zip(gp, r.best_point):
        assert abs(a - b) <= param_atol * max(1.0, abs(b)), (gp, r.best_point)


def ref_anneal_static(ref, surface, slice, schedule):
    """The reference's minimize on the reference's static objective with the
    default box and the ATM start: the run calibrate_static_T1 makes
    (calibration.cpp:289-306), with its temperature trace."""
    from oracles import atm_vol_guess

    lo, hi = [1e-4, 0.0, 1e-4, -1.0], [2.0, 1.0, 10.0, 1.0]
    start = [atm_vol_guess(surface, slice), 1.0, 0.5, -0.3]
    schedule.omp_threads = ref.max_threads()
    return ref.minimize_cost(pkg.MODEL_STATIC, surface, slice, lo, hi, schedule, start)


@pytest.mark.parametrize("slice", [0, 1, 2, 3])
def test_c2_shape_first_levels_match_reference(engine, ref, fx_surface, slice):
    import bench

    s = bench.c2_schedule(1, max_evals=2 * 10 ** 7 + 1)
    g = engine.calibrate_static_T1(fx_surface, slice, None, s, None, trace=True)
    r = ref_anneal_static(ref, fx_surface, slice, s)
    assert g.evals == r.evals == 2 * 10 ** 7 + 1 and len(r.temperature_trace) == 2
    assert_same_anneal(g, r)
    # and the report rows against the reference's calibrate_static_T1 itself
    rep = ref.calibrate_static_T1(fx_surface, slice, None, s, None)
    assert rep.evals == g.evals and abs(rep.final_cost - g.final_cost) <= 1e-12 * rep.final_cost
    for a, b in zip(g.rows, rep.rows):
        assert a.strike == b.strike and abs(a.model - b.model) <= 1e-9 * abs(b.model)


@pytest.mark.slow
def test_c2_full_run_matches_reference(engine, ref, fx_surface):
    """The whole C2 calibration of the 3m slice: 412 levels, 4.12e9 evals."""
    import bench

    s = bench.c2_schedule(1)
    g = engine.calibrate_static_T1(fx_surface, 0, None, s, None, trace=True)
    r = ref_anneal_static(ref, fx_surface, 0, s)
    assert g.evals == r.evals == 100_000 * 100 * bench.LEVELS_C1 + 1
    assert_same_anneal(g, r)


def test_c3_beta_free_acceptance_schedule(engine, ref, fx_surface):
    s = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=32, t_min=1e-7, seed=1)
    g = engine.calibrate_dynamic_case1_T1(fx_surface, None, s, None)
    s.omp_threads = ref.max_threads()
    r = ref.calibrate_dynamic_case1_T1(fx_surface, None, s, None)
    assert g.evals == r.evals == 1_000_001
    assert_same_run_report(g, r)


def test_c3_beta_free_full_width_level(engine, ref, fx_surface):
    s = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=12_500, groups=8, t_min=1e-7,
                              seed=1, max_evals=10 ** 7 + 1)
    g = engine.calibrate_dynamic_case1_T1(fx_surface, None, s, None)
    s.omp_threads = ref.max_threads()
    r = ref.calibrate_dynamic_case1_T1(fx_surface, None, s, None)
    assert g.evals == r.evals == 10 ** 7 + 1
    assert_same_run_report(g, r)


def assert_same_run_report(g, r):
    assert g.evals == r.evals
    assert abs(g.final_cost - r.final_cost) <= 1e-11 * abs(r.final_cost), (g.final_cost, r.final_cost)
    for k in r.params:
        assert abs(g.params[k] - r.params[k]) <= 1e-8 * max(1.0, abs(r.params[k])), (k, g.params[k], r.params[k])
    for a, b in zip(g.rows, r.rows):
        assert abs(a.model - b.model) <= 1e-9 * abs(b.model)


def c5_one_step(chains, paths):
    import bench

    surf = pkg.parse_surface(os.path.join(DATA, "synth20x30.csv"))
    sch = pkg.AnnealingSchedule(t0=2.0, cooling=0.5, chain_length=1, workers=chains // 8, groups=8, t_min=1.5,
                                seed=1, max_evals=10 ** 12)
    plan = pkg.SimulationPlan(num_paths=paths, dt=1 / 250, seed=1, rng="xoshiro")
    return surf, sch, plan, bench.c5_bounds()


@pytest.mark.slow
def test_c5_per_gpu_step_matches_reference(engine, ref):
    """125,000 chains (workers 15625 x groups 8), one SA step, one path per
    candidate on all 20 slices (13130 steps): every candidate's feasibility,
    MC cost and Metropolis decision enter the merge."""
    surf, sch, plan, box = c5_one_step(125_000, 1)
    g = engine.calibrate_case2_T2(surf, box, sch, plan, None)
    sch.omp_threads = ref.max_threads()
    r = ref.calibrate_case2_T2(surf, box, sch, plan, None)
    assert g.evals == r.evals and g.evals > 100_000
    assert abs(g.final_cost - r.final_cost) <= 1e-10 * abs(r.final_cost), (g.final_cost, r.final_cost)
    for k in r.params:
        assert abs(g.params[k] - r.params[k]) <= 1e-9 * max(1.0, abs(r.params[k])), k


C5_DEFAULT_BOX_CHILD = r"""
import os, sys
sys.path[:0] = [{root!r}, os.path.join({root!r}, "tests")]
import paper_2407_20713_b200 as pkg
from oracles import Ref
surf = pkg.parse_surface(os.path.join({root!r}, "tests", "data", "synth20x30.csv"))
sch = pkg.AnnealingSchedule(t0=2.0, cooling=0.5, chain_length=1, workers=2000 // 8, groups=8, t_min=1.5,
                            seed=1, max_evals=10 ** 12)
plan = pkg.SimulationPlan(num_paths=2, dt=1 / 250, seed=1, rng="xoshiro")
Ref().calibrate_case2_T2(surf, None, sch, plan, None)
print("REFERENCE-RETURNED")
"""


def test_c5_default_box_reference_aborts_engine_completes(engine, ref):
    """In the default Case II box (calibration.cpp:46-60) at T = t0 the
    proposals include exploding dynamics.  The reference's running product
    F *= exp(...) (mc.cpp:97-103) overflows on some paths, its
    runtime_error("mc: non-finite path value ...", mc.cpp:137-138) escapes
    the OpenMP region and the process terminates.  The engine carries the
    path in log space (F_T = F0 e^x), where such an excursion
    stays finite, so the same call completes with a finite cost (the
    candidate's absurd price makes it a rejected move).  A deliberate
    difference: there is no reference result to compare."""
    child = subprocess.run([sys.executable, "-c", C5_DEFAULT_BOX_CHILD.format(root=ROOT)],
                           capture_output=True, text=True, timeout=600)
    assert "REFERENCE-RETURNED" not in child.stdout
    assert "non-finite path value" in child.stderr
    surf, sch, plan, _ = c5_one_step(2000, 2)
    g = engine.calibrate_case2_T2(surf, None, sch, plan, None)
    assert np.isfinite(g.final_cost) and g.evals > 100


# ---- Case II feasibility (analytics.cpp:145-175), directly ----
EQ_CASE2 = [0.296790, 1.0, -0.360610, 15.0, -0.715716, 0.000100, -8.969205, 0.847244, 15.0, 15.0]
FX_CASE2 = [0.154037, 1.0, -0.693682, 0.345973, -0.200342, 7.541424, -0.992551, 0.339807, 0.0, 150.0]


def test_case2_feasible_batch_matches_reference(engine, ref):
    """sabr_case2_feasible_batch vs CaseIIParams::validate on the grid rule:
    random vectors in and around the default box, the two published fits at
    horizons 0.05..5 (the equity fit has rho(0+) = -1.076 and passes only
    because the first grid node lies past the violating interval), and
    vectors on the 1e-9 rho tolerance and the stationary-point boundary."""
    rng = np.random.default_rng(11)
    lo = np.array([1e-4, 0, -1, -15, -1, 1e-4, -15, -1, 0, 0])
    hi = np.array([2, 1, 1, 15, 1, 10, 15, 1, 150, 150])
    P = lo + (hi - lo) * rng.random((20000, 10))
    P[:, 3] *= rng.random(len(P)) ** 3
    P[:, 6] *= rng.random(len(P)) ** 3
    H = rng.choice([0.25, 0.5, 1.0, 2.0, 5.0], len(P))
    rows = [np.column_stack([P, H])]
    horizons = np.concatenate([np.linspace(0.05, 5.0, 100), [0.25, 0.5, 0.75, 0.9, 0.95, 0.96, 0.97, 1.0, 2.0]])
    for fit in (EQ_CASE2, FX_CASE2):
        rows.append(np.array([fit + [h] for h in horizons]))
    # rho(t) = (rho0 + q t) e^{-a t} + d exactly on / beside the 1 + 1e-9 edge at t = 0+
    edge = []
    for d in (1e-9, 0.5e-9, 2e-9, -1e-9, -2e-9):
        edge.append([0.3, 0.5, 1.0, 0.0, d, 0.5, 0.0, 0.0, 0.0, 0.0, 1.0])
        edge.append([0.3, 0.5, -1.0, 0.0, -d, 0.5, 0.0, 0.0, 0.0, 0.0, 1.0])
    rows.append(np.array(edge))
    Q = np.vstack(rows)
    got = engine.case2_feasible_batch(Q)
    want = ref.case2_feasible(Q)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, Q[bad[:5]]
    # the equity fit: infeasible at short horizons, feasible from ~0.96 on
    eq = np.array([EQ_CASE2 + [h] for h in (0.25, 0.5, 2.0)])
    assert list(ref.case2_feasible(eq)) == list(engine.case2_feasible_batch(eq))
    print("feasible fraction", want.mean(), "equity fit at 0.25/0.5/2:", list(ref.case2_feasible(eq)))
