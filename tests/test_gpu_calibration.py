"""calibrate_* through the C-ABI against the compiled reference's own
calibrate_* (proj/src/calibration.cpp) and its unit tests
(proj/tests/test_calibration.cpp)."""
import os

import numpy as np
import pytest

import paper_2407_20713_b200 as pkg

pytestmark = pytest.mark.gpu


def c1_schedule(seed):
    # acceptance.cpp:318-323
    return pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=32, t_min=1e-7, seed=seed)


def close_reports(g, r, rtol=1e-10):
    assert g.model == r.model and g.technique == r.technique and g.quantity == r.quantity
    assert g.evals == r.evals
    assert abs(g.final_cost - r.final_cost) <= rtol * abs(r.final_cost)
    assert g.params.keys() == r.params.keys()
    for k in r.params:
        assert abs(g.params[k] - r.params[k]) <= 1e-7 * max(1.0, abs(r.params[k])), (k, g.params[k], r.params[k])
    assert len(g.rows) == len(r.rows)
    for a, b in zip(g.rows, r.rows):
        assert a.maturity == b.maturity and a.strike == b.strike and a.market == b.market
        assert abs(a.model - b.model) <= 1e-9 * abs(b.model)
    assert abs(g.mean_rel_error - r.mean_rel_error) <= 1e-7 * r.mean_rel_error


@pytest.mark.parametrize("seed", [1, 2])
def test_static_T1_matches_reference(engine, ref, eq_surface, seed):
    s = c1_schedule(seed)
    g = engine.calibrate_static_T1(eq_surface, 0, None, s, None)
    r = ref.calibrate_static_T1(eq_surface, 0, None, s, None)
    close_reports(g, r)
    assert g.seed == seed


def test_static_T1_slices_match_one_slice_calls(engine, fx_surface):
    """sabr_calibrate_static_T1_slices runs each slice's annealer on its own
    stream and host thread; every report must equal the one-slice call's, bit
    for bit (parameters, cost, evals, rows, temperature trace), for all slices,
    a reordered subset, and repeated calls (the child contexts are reused)."""
    s = pkg.AnnealingSchedule(t0=2.0, cooling=0.8, chain_length=20, workers=500, groups=4, t_min=1e-3, seed=3)
    single = [engine.calibrate_static_T1(fx_surface, i, None, s, None, trace=True)
              for i in range(len(fx_surface.slices))]
    for sel in (None, [2, 0], [3]):
        for _ in range(2):
            multi = engine.calibrate_static_T1_slices(fx_surface, sel, None, s, None, trace=True)
            idx = list(range(len(fx_surface.slices))) if sel is None else sel
            assert len(multi) == len(idx)
            for i, m in zip(idx, multi):
                g = single[i]
                assert m.evals == g.evals and m.final_cost == g.final_cost and m.params == g.params
                assert m.temperature_trace == g.temperature_trace
                assert [(r.strike, r.model) for r in m.rows] == [(r.strike, r.model) for r in g.rows]
    # more slices than side-by-side streams (8): each stream runs its share in order
    many = list(range(len(fx_surface.slices))) * 3
    for i, m in enumerate(engine.calibrate_static_T1_slices(fx_surface, many, None, s, None, trace=True)):
        g = single[i % len(fx_surface.slices)]
        assert m.evals == g.evals and m.final_cost == g.final_cost and m.params == g.params
        assert m.temperature_trace == g.temperature_trace
    with pytest.raises(pkg.OutOfRangeError):
        engine.calibrate_static_T1_slices(fx_surface, [0, 9], None, s, None)
    assert engine.calibrate_static_T1_slices(fx_surface, [], None, s, None) == []


def test_static_T1_fixed_and_bounds(engine, ref, fx_surface):
    s = pkg.AnnealingSchedule(t0=1.0, cooling=0.8, chain_length=10, workers=4, t_min=1e-2, seed=1)
    g = engine.calibrate_static_T1(fx_surface, 0, {"nu": (0.01, 3.0)}, s, {"beta": 0.75, "rho": -0.4})
    r = ref.calibrate_static_T1(fx_surface, 0, {"nu": (0.01, 3.0)}, s, {"beta": 0.75, "rho": -0.4})
    close_reports(g, r)
    assert g.params["beta"] == 0.75 and g.params["rho"] == -0.4


def test_evaluation_only_mode(engine, ref, eq_surface):
    fixed = {"alpha": 0.289271, "beta": 1.0, "nu": 0.308560, "rho": -0.999729}
    g = engine.calibrate_static_T1(eq_surface, 2, None, pkg.AnnealingSchedule(seed=99), fixed)
    r = ref.calibrate_static_T1(eq_surface, 2, None, pkg.AnnealingSchedule(seed=99), fixed)
    assert g.evals == 1 and len(g.rows) == 21
    close_reports(g, r)


def test_case1_T1_matches_reference(engine, ref, fx_surface):
    s = pkg.AnnealingSchedule(t0=2.0, cooling=0.9, chain_length=50, workers=32, t_min=1e-5, seed=1)
    g = engine.calibrate_dynamic_case1_T1(fx_surface, None, s, {"beta": 1.0})
    r = ref.calibrate_dynamic_case1_T1(fx_surface, None, s, {"beta": 1.0})
    close_reports(g, r)


def test_case1_evaluation_published_fit(engine, ref, eq_surface):
    p = pkg.CaseIParams(0.294722, 1.0, -1.0, 0.388539, 0.001, 0.131466)
    g = engine.evaluate_case1(eq_surface, p)
    assert len(g.rows) == 84 and g.quantity == "vol"
    assert abs(g.mean_rel_error - 2.073025e-2) <= 2.5e-2 * 2.073025e-2
    assert g.max_rel_error < 0.10
    close_reports_eval = ref.evaluate_case1(eq_surface, p)
    assert abs(g.final_cost - close_reports_eval.final_cost) <= 1e-12 * close_reports_eval.final_cost


def test_errors_map_to_reference_exceptions(engine, fx_surface):
    s = pkg.AnnealingSchedule()
    with pytest.raises(pkg.DomainError):
        engine.calibrate_static_T1(fx_surface, 0, {"alpha": (2.0, 1.0)}, s, None)
    with pytest.raises(pkg.DomainError):
        engine.calibrate_static_T1(fx_surface, 0, {"gamma": (0.0, 1.0)}, s, None)
    with pytest.raises(pkg.DomainError):
        engine.calibrate_static_T1(fx_surface, 0, None, s, {"gamma": 0.5})
    with pytest.raises(pkg.OutOfRangeError):
        engine.calibrate_static_T1(fx_surface, 9, None, s, None)
    one = pkg.VolSurface(fx_surface.spot, [fx_surface.slices[0]])
    with pytest.raises(pkg.DomainError):
        engine.calibrate_dynamic_case1_T1(one, None, s, None)


def test_case2_T2_matches_reference(engine, ref, eq_surface):
    """calibrate_case2_T2 end to end (no reference test exists for it: the
    reference itself is the oracle here).  C4 shape at small scale: the T = 1
    equity slice, dynamics pinned static, reference xoshiro streams."""
    surf = pkg.VolSurface(eq_surface.spot, [eq_surface.slices[2]])
    fixed = {"a": 0.0, "b": 0.0, "q_rho": 0.0, "q_nu": 0.0, "d_rho": 0.0, "d_nu": 0.0, "beta": 1.0}
    s = pkg.AnnealingSchedule(t0=2.0, cooling=0.5, chain_length=4, workers=6, t_min=0.2, seed=3)
    plan = pkg.SimulationPlan(num_paths=2048, seed=1)
    g = engine.calibrate_case2_T2(surf, None, s, plan, fixed)
    r = ref.calibrate_case2_T2(surf, None, s, plan, fixed)
    assert g.evals == r.evals
    assert abs(g.final_cost - r.final_cost) <= 1e-9 * r.final_cost
    for k in r.params:
        assert abs(g.params[k] - r.params[k]) <= 1e-7 * max(1.0, abs(r.params[k])), k
    for a, b in zip(g.rows, r.rows):
        assert abs(a.model - b.model) <= 1e-9 * abs(b.model)


def test_case2_T2_full_case2_synthetic_surface(engine, ref):
    """The C5 shape at small scale: every Case II parameter free (beta too),
    the 20-maturity x 30-strike synthetic surface, reference xoshiro streams,
    box narrowed around the published FX fit as in bench.py (c5_bounds)."""
    import bench

    surf = pkg.parse_surface(os.path.join(os.path.dirname(__file__), "data", "synth20x30.csv"))
    s = pkg.AnnealingSchedule(t0=2.0, cooling=0.5, chain_length=2, workers=4, t_min=0.9, seed=4)
    plan = pkg.SimulationPlan(num_paths=256, seed=2)
    g = engine.calibrate_case2_T2(surf, bench.c5_bounds(), s, plan, None)
    r = ref.calibrate_case2_T2(surf, bench.c5_bounds(), s, plan, None)
    assert g.evals == r.evals
    assert abs(g.final_cost - r.final_cost) <= 1e-9 * r.final_cost
    for k in r.params:
        assert abs(g.params[k] - r.params[k]) <= 1e-7 * max(1.0, abs(r.params[k])), k
    assert len(g.rows) == len(r.rows) == 600
    for a, b in zip(g.rows, r.rows):
        assert abs(a.model - b.model) <= 1e-9 * abs(b.model)


def test_case2_T2_fp32_fast_path(engine, eq_surface):
    """The FP32 MC objective drives the same annealer: the same proposals are
    evaluated (evals depend on feasibility only) and the calibrated cost stays
    within the FP32 price tolerance of the FP64 run's neighbourhood."""
    surf = pkg.VolSurface(eq_surface.spot, [eq_surface.slices[2]])
    fixed = {"a": 0.0, "b": 0.0, "q_rho": 0.0, "q_nu": 0.0, "d_rho": 0.0, "d_nu": 0.0, "beta": 1.0}
    s = pkg.AnnealingSchedule(t0=2.0, cooling=0.5, chain_length=4, workers=32, t_min=0.2, seed=3)
    p64 = pkg.SimulationPlan(num_paths=1 << 14, seed=1)
    p32 = pkg.SimulationPlan(num_paths=1 << 14, seed=1, precision="fp32")
    a = engine.calibrate_case2_T2(surf, None, s, p64, fixed)
    b = engine.calibrate_case2_T2(surf, None, s, p32, fixed)
    assert a.evals == b.evals
    assert abs(a.final_cost - b.final_cost) <= 1e-2 * a.final_cost


def test_case2_formula_matches_reference(engine, ref, fx_surface):
    """calibrate_case2_formula (calibration.cpp:483-534) end to end."""
    s = pkg.AnnealingSchedule(t0=2.0, cooling=0.5, chain_length=8, workers=16, t_min=0.05, seed=2)
    g = engine.calibrate_case2_formula(fx_surface, None, s, {"beta": 1.0})
    r = ref.calibrate_case2_formula(fx_surface, None, s, {"beta": 1.0})
    assert g.model == "case2" and g.technique == "T_I" and g.quantity == "price" and not g.rows
    assert g.evals == r.evals
    assert abs(g.final_cost - r.final_cost) <= 1e-9 * r.final_cost
    for k in r.params:
        assert abs(g.params[k] - r.params[k]) <= 1e-7 * max(1.0, abs(r.params[k])), k


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("case", ["c4_shape", "c5_shape"])
def test_case2_T2_candidate_block_invariance(engine, eq_surface, precision, case, monkeypatch):
    """The MC tile kernels simulate CB candidates per thread (SABR_MC_CB: 1, 2,
    4, 8, 16; the FP32 kernel runs them as packed FP32x2 pairs reading the
    pair-interleaved coefficient rows, CB = 1 a half-idle pair on the plain
    rows).  A candidate's arithmetic, its payoff column sums and the tile
    reduction do not depend on CB, so the whole T_II report (evals, trace,
    parameters, cost) must be bit-identical for every CB.  c4_shape: static
    dynamics on one 250-step slice (the time-invariant-row kernels); c5_shape:
    full Case II on the 20x30 synthetic surface (time-varying rows)."""
    import bench

    if case == "c4_shape":
        surf = pkg.VolSurface(eq_surface.spot, [eq_surface.slices[2]])
        fixed = {"a": 0.0, "b": 0.0, "q_rho": 0.0, "q_nu": 0.0, "d_rho": 0.0, "d_nu": 0.0, "beta": 1.0}
        bounds = None
        s = pkg.AnnealingSchedule(t0=2.0, cooling=0.5, chain_length=3, workers=40, t_min=0.4, seed=5)
        plan = pkg.SimulationPlan(num_paths=3000, seed=1, precision=precision)
    else:
        surf = pkg.parse_surface(os.path.join(os.path.dirname(__file__), "data", "synth20x30.csv"))
        fixed, bounds = None, bench.c5_bounds()
        s = pkg.AnnealingSchedule(t0=2.0, cooling=0.5, chain_length=2, workers=24, t_min=0.9, seed=4)
        plan = pkg.SimulationPlan(num_paths=300, seed=2, precision=precision)
    reps = {}
    for cb in (1, 2, 4, 8, 16):
        monkeypatch.setenv("SABR_MC_CB", str(cb))
        reps[cb] = engine.calibrate_case2_T2(surf, bounds, s, plan, fixed)
    a = reps[8]
    for cb, b in reps.items():
        assert b.evals == a.evals, cb
        assert b.final_cost == a.final_cost, (cb, b.final_cost, a.final_cost)
        assert b.params == a.params, cb
        assert b.temperature_trace == a.temperature_trace, cb


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_case2_T2_pdl_chain_matches_serialised_launches(engine, eq_surface, precision, monkeypatch):
    """The kernels of a T_II step (propose, compact, coefficients, MC tiles,
    reduction, finish) are chained by programmatic dependent launch (pdl.cuh):
    a kernel may start its stream-independent set-up while its predecessor
    runs and waits for it in-kernel.  SABR_T2_PDL=0 launches them fully
    serialised; the report must be bit-identical."""
    surf = pkg.VolSurface(eq_surface.spot, [eq_surface.slices[2]])
    fixed = {"a": 0.0, "b": 0.0, "q_rho": 0.0, "q_nu": 0.0, "d_rho": 0.0, "d_nu": 0.0, "beta": 1.0}
    s = pkg.AnnealingSchedule(t0=2.0, cooling=0.5, chain_length=3, workers=40, t_min=0.4, seed=6)
    plan = pkg.SimulationPlan(num_paths=2000, seed=3, precision=precision)
    reps = {}
    for v in ("0", "1"):
        monkeypatch.setenv("SABR_T2_PDL", v)
        reps[v] = engine.calibrate_case2_T2(surf, None, s, plan, fixed)
    a, b = reps["0"], reps["1"]
    assert b.evals == a.evals
    assert b.final_cost == a.final_cost
    assert b.params == a.params
    assert b.temperature_trace == a.temperature_trace


def test_case2_T2_wide_slice_matches_reference(engine, ref):
    """A slice of 400 quotes: the tile kernel's payoff accumulators outgrow
    shared memory at 8 or 16 candidates per thread, so the engine drops to the
    largest block that fits (kernels_mc.cu mc_max_cand_block); results as the
    reference's."""
    K = np.linspace(60.0, 140.0, 400)
    quotes = [pkg.VolQuote(float(k), float(0.2 + 0.1 * (k / 100.0 - 1.0) ** 2)) for k in K]
    surf = pkg.VolSurface(100.0, [pkg.VolSlice(1.0, 0.01, 0.0, quotes)])
    fixed = {"a": 0.0, "b": 0.0, "q_rho": 0.0, "q_nu": 0.0, "d_rho": 0.0, "d_nu": 0.0, "beta": 1.0}
    s = pkg.AnnealingSchedule(t0=2.0, cooling=0.5, chain_length=2, workers=16, t_min=0.9, seed=6)
    plan = pkg.SimulationPlan(num_paths=512, seed=3)
    g = engine.calibrate_case2_T2(surf, None, s, plan, fixed)
    r = ref.calibrate_case2_T2(surf, None, s, plan, fixed)
    assert g.evals == r.evals
    assert abs(g.final_cost - r.final_cost) <= 1e-9 * r.final_cost
    for k in r.params:
        assert abs(g.params[k] - r.params[k]) <= 1e-7 * max(1.0, abs(r.params[k])), k
