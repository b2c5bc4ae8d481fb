"""Acceptance criterion c10 (proj/tests/acceptance.cpp:317-414) on the GPU:
end-to-end calibration quality on both market surfaces.

* T_I: calibrate_dynamic_case1_T1 with beta = 1 fixed, the C1 schedule
  (t0 2, cooling 0.96, L 100, 32 workers, t_min 1e-7), seeds 1..3 until the
  cap is met: mean relative vol error <= 2.6e-2 (equity) / 3.1e-2 (fx).
* "T_II": calibrate_case2_formula (L 60) then evaluate_case2_prices at 2^16
  paths, seed = the schedule seed: mean relative price error <= 2.5e-2 /
  3.0e-2 (acceptance.cpp:341-366).

The reference artifact's own run (proj/test_output.txt:36-39, seed 1 met
every cap) printed 2.0772e-02 / 2.4340e-02 (T_I, 3 s each on its host) and
1.5620e-02 / 2.8509e-02 (T_II, 253 s / 218 s); the same trajectories on the
GPU reproduce those four numbers to the printed digits.

The worker-scaling half of c10 (8-vs-1 OpenMP threads) has no device analogue;
the rank-count independence of the results is tests/test_gpu_multirank_engine.py."""
import pytest

import paper_2407_20713_b200 as pkg

pytestmark = pytest.mark.gpu


def best_over_seeds(run, cap):
    best = float("inf")
    for seed in (1, 2, 3):
        best = min(best, run(seed))
        if best <= cap:
            break
    return best


@pytest.mark.parametrize("fixture,cap,printed", [("eq_surface", 2.6e-2, "2.0772e-02"),
                                                 ("fx_surface", 3.1e-2, "2.4340e-02")])
def test_c10_t1_case1(engine, request, fixture, cap, printed):
    surface = request.getfixturevalue(fixture)

    def run(seed):
        s = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=32, t_min=1e-7, seed=seed)
        return engine.calibrate_dynamic_case1_T1(surface, None, s, {"beta": 1.0}).mean_rel_error

    best = best_over_seeds(run, cap)
    print(f"c10 T_I {fixture}: mean rel vol error {best:.4e} (cap {cap})")
    assert best <= cap and f"{best:.4e}" == printed


@pytest.mark.parametrize("fixture,cap,printed", [("eq_surface", 2.5e-2, "1.5620e-02"),
                                                 ("fx_surface", 3.0e-2, "2.8509e-02")])
def test_c10_t2_formula_then_mc(engine, request, fixture, cap, printed):
    surface = request.getfixturevalue(fixture)
    names = ["alpha", "beta", "rho0", "q_rho", "d_rho", "nu0", "q_nu", "d_nu", "a", "b"]

    def run(seed):
        s = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=60, workers=32, t_min=1e-7, seed=seed)
        rep = engine.calibrate_case2_formula(surface, None, s, {"beta": 1.0})
        p = pkg.CaseIIParams(*[rep.params[k] for k in names], surface.slices[-1].maturity)
        ev = engine.evaluate_case2_prices(surface, p, pkg.SimulationPlan(num_paths=1 << 16, seed=seed))
        return ev.mean_rel_error

    best = best_over_seeds(run, cap)
    print(f"c10 T_II {fixture}: mean rel price error {best:.4e} (cap {cap})")
    assert best <= cap and f"{best:.4e}" == printed
