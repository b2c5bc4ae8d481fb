"""How often does the engine's annealer trajectory leave the reference's?

The default objective is the factored slice cost ||R v||^2,
which agrees with the reference's per-quote sum to ~1e-14 relative, not bit
for bit, and the device exp/log/pow differ from glibc's in the last bit.  A
Metropolis comparison (fy <= fx, u < exp(-(fy-fx)/T)) can therefore flip on a
near-tie, after which the two runs are different (equally valid) annealer
trajectories.  This test measures the rate on randomized surfaces and seeds
(static Hagan T_I, the C1-style 32-chain schedule shortened to ~1e5 evals per
run), reports it, and bounds it.  A run "diverges" when its evals, trace
length or any trace value (beyond 1e-10 relative) differ from the
reference's."""
import numpy as np
import pytest

import paper_2407_20713_b200 as pkg

pytestmark = pytest.mark.gpu

N_SURFACES = 24
SEEDS = (1, 2)


def random_surface(rng, orc):
    spot = float(rng.uniform(0.5, 5000.0))
    T = float(rng.uniform(0.1, 3.0))
    r, y = float(rng.uniform(0.0, 0.05)), float(rng.uniform(0.0, 0.04))
    m = int(rng.integers(5, 41))
    f = spot * np.exp((r - y) * T)
    K = np.sort(f * np.exp(rng.uniform(-0.5, 0.5, m)))
    K = np.unique(K)
    p = [float(rng.uniform(0.05, 0.6)) * f ** (1 - 0.7), 0.7, float(rng.uniform(0.1, 1.5)),
         float(rng.uniform(-0.8, 0.3))]
    vols = []
    for k in K:
        v = orc.static_vol(p, float(k), f, T)
        vols.append(v * (1.0 + 0.01 * rng.standard_normal()))
    vols = [max(v, 1e-3) for v in vols]
    qs = [pkg.VolQuote(float(k), float(v)) for k, v in zip(K, vols)]
    return pkg.VolSurface(spot, [pkg.VolSlice(T, r, y, qs)])


def test_trajectory_divergence_rate(engine, ref, orc):
    from oracles import atm_vol_guess

    rng = np.random.default_rng(2026)
    runs, diverged = 0, []
    for i in range(N_SURFACES):
        surf = random_surface(rng, orc)
        for seed in SEEDS:
            s = pkg.AnnealingSchedule(t0=2.0, cooling=0.9, chain_length=50, workers=32, t_min=1e-6, seed=seed)
            g = engine.calibrate_static_T1(surf, 0, None, s, None, trace=True)
            s.omp_threads = ref.max_threads()
            lo, hi = [1e-4, 0.0, 1e-4, -1.0], [2.0, 1.0, 10.0, 1.0]
            start = [atm_vol_guess(surf, 0), 1.0, 0.5, -0.3]
            r = ref.minimize_cost(pkg.MODEL_STATIC, surf, 0, lo, hi, s, start)
            runs += 1
            same = g.evals == r.evals and len(g.temperature_trace) == len(r.temperature_trace)
            if same:
                for (_, a), (_, b) in zip(g.temperature_trace, r.temperature_trace):
                    if abs(a - b) > 1e-10 * max(abs(b), 1e-300):
                        same = False
                        break
            if not same:
                diverged.append((i, seed, g.evals, r.evals, g.final_cost, r.best_value))
            else:
                # identical decisions: the same optimum to the cost tolerance
                assert abs(g.final_cost - r.best_value) <= 1e-10 * abs(r.best_value)
    rate = len(diverged) / runs
    print(f"trajectory divergence: {len(diverged)} of {runs} runs ({rate:.1%}); {diverged}")
    # a divergent run is a different trajectory of the same annealer, not a
    # worse fit: its optimum stays within a few percent of the reference's
    for (_, _, _, _, gc, rc) in diverged:
        assert gc <= 1.5 * rc + 1e-12
    assert rate <= 0.10
