"""The BASELINE.json workloads at their full sizes, through properties that do
not need a CPU run of the same size (the reference would need minutes to hours
per case):

* C2 (1e5 chains, 412 levels, 4.12e9 evals per slice): the run is
  deterministic, the eval count is exactly the schedule's, the temperature
  trace is non-increasing (annealer.cpp:141-160 only ever lowers the
  incumbent), the reported optimum lies in the box and its cost recomputed by
  the batched objective equals the reported cost, and the report rows are the
  model vols at that point.
* C4 (1e5 paths x 250 steps): the MC objective (case2_mc_cost) at two
  points equals the reference's at the same plan (same xoshiro streams) to
  1e-11.
* C5 (20 x 30 surface, 4096 paths): one full-surface MC cost equals the
  reference's to 1e-11."""
import os

import numpy as np
import pytest

import paper_2407_20713_b200 as pkg

pytestmark = pytest.mark.gpu

DATA = os.path.join(os.path.dirname(__file__), "data")


def test_c2_full_size_properties(engine, fx_surface):
    import bench

    sch = bench.c2_schedule(1)
    a = engine.calibrate_static_T1(fx_surface, 0, None, sch, None, trace=True)
    b = engine.calibrate_static_T1(fx_surface, 0, None, sch, None, trace=True)
    assert a.final_cost == b.final_cost and a.params == b.params and a.temperature_trace == b.temperature_trace
    assert a.evals == 100_000 * 100 * bench.LEVELS_C1 + 1
    f = [v for _, v in a.temperature_trace]
    assert len(f) == bench.LEVELS_C1 and all(x >= y for x, y in zip(f, f[1:]))
    p = [a.params[k] for k in ("alpha", "beta", "nu", "rho")]
    for v, (lo, hi) in zip(p, [(1e-4, 2.0), (0.0, 1.0), (1e-4, 10.0), (-1.0, 1.0)]):
        assert lo <= v <= hi
    c = engine.cost_batch(pkg.MODEL_STATIC, fx_surface, np.array([p]), slice=0)[0]
    assert c == a.final_cost
    vols = engine.implied_vol_batch(pkg.MODEL_STATIC, fx_surface, np.array([p]), slice=0)[0]
    assert [r.model for r in a.rows] == list(vols)
    assert a.final_cost <= f[-1]


def test_c4_full_size_mc_cost_matches_reference(engine, ref, eq_surface):
    surf = pkg.VolSurface(eq_surface.spot, [eq_surface.slices[2]])
    plan = pkg.SimulationPlan(num_paths=100_000, dt=1 / 250, seed=1)
    P = np.array([[0.30, 1.0, -0.45, 0.0, 0.0, 0.9, 0.0, 0.0, 0.0, 0.0, 1.0],
                  [0.25, 1.0, -0.60, 0.0, 0.0, 1.4, 0.0, 0.0, 0.0, 0.0, 1.0]])
    got = engine.cost_batch(pkg.MODEL_CASE2, surf, P, plan=plan)
    want = ref.cost_case2_mc(surf, P, plan)
    assert np.max(np.abs(got - want) / want) < 1e-11


def test_c5_full_surface_mc_cost_matches_reference(engine, ref):
    surf = pkg.parse_surface(os.path.join(DATA, "synth20x30.csv"))
    plan = pkg.SimulationPlan(num_paths=4096, dt=1 / 250, seed=1)
    P = np.array([[0.154037, 1.0, -0.693682, 0.345973, -0.200342, 7.541424, -0.992551, 0.339807, 0.0, 150.0, 5.0]])
    got = engine.cost_batch(pkg.MODEL_CASE2, surf, P, plan=plan)
    want = ref.cost_case2_mc(surf, P, plan)
    assert np.max(np.abs(got - want) / want) < 1e-11
