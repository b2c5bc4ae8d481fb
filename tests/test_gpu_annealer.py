"""The reference annealer's own unit tests (proj/tests/test_annealer.cpp) run
against the GPU driver on the same closed-form objectives, plus trajectory
parity with the restated annealer (oracle/sabr_oracle.c:orc_minimize): the
chain streams are keyed exactly as annealer.cpp:114-115, so evals, the
temperature trace and the best point coincide."""
import math

import numpy as np
import pytest

import paper_2407_20713_b200 as pkg
from paper_2407_20713_b200 import _abi as A

pytestmark = pytest.mark.gpu


def quick(**kw):
    s = pkg.AnnealingSchedule(t0=5.0, cooling=0.9, chain_length=40, workers=8, t_min=1e-6, seed=1)
    for k, v in kw.items():
        setattr(s, k, v)
    return s


def test_quadratic_bowl(engine):
    r = engine.minimize_builtin(A.OBJ_BOWL3, [-5] * 3, [5] * 3, quick(), [0, 0, 0])
    assert r.best_value < 1e-6
    assert abs(r.best_point[0] - 1.2) < 1e-2 and abs(r.best_point[1] + 0.7) < 1e-2
    assert abs(r.best_point[2] - 3.4) < 1e-2


def test_rosenbrock_most_seeds(engine):
    good = 0
    for seed in range(10):
        r = engine.minimize_builtin(A.OBJ_ROSENBROCK4, [-2] * 4, [2] * 4,
                                    quick(seed=seed, chain_length=120, t_min=1e-8), [-1, 1, -1, 1])
        good += r.best_value < 1e-2
    assert good >= 8


def test_budget_respected(engine):
    s = quick(max_evals=500)
    r = engine.minimize_builtin(A.OBJ_SQUARE1, [-1], [1], s, [0.5])
    assert r.evals <= s.max_evals + s.workers * s.groups


def test_trace_monotone(engine):
    r = engine.minimize_builtin(A.OBJ_COSBOWL2, [-3, -3], [3, 3], quick(), [2, -2])
    tr = [f for _, f in r.temperature_trace]
    assert all(b <= a for a, b in zip(tr, tr[1:]))
    assert r.best_value <= tr[-1]


def test_infeasible_never_evaluated(engine):
    r = engine.minimize_builtin(A.OBJ_CORNER2, [-2, -2], [2, 2], quick(), [0, 0], predicate=A.PRED_SUM_LE_1)
    assert abs(r.best_value - 4.5) <= 4.5e-3
    assert r.best_point[0] + r.best_point[1] <= 1.0


def test_nan_is_infinitely_bad(engine):
    r = engine.minimize_builtin(A.OBJ_NANRIGHT1, [-2], [2], quick(), [0])
    assert math.isfinite(r.best_value) and abs(r.best_point[0] + 1) < 1e-2


def test_schedule_validation(engine):
    for bad in (quick(cooling=1.1), quick(t0=0.0), quick(workers=0)):
        with pytest.raises(pkg.DomainError):
            engine.minimize_builtin(A.OBJ_SQUARE1, [-1], [1], bad, [0.5])
    with pytest.raises(pkg.DomainError):
        engine.minimize_builtin(A.OBJ_SQUARE1, [2], [1], quick(), [1.5])


@pytest.mark.parametrize("obj,lo,hi,start,pred", [
    (A.OBJ_BOWL3, [-5] * 3, [5] * 3, [0, 0, 0], 0),
    (A.OBJ_SINQUAD2, [-5, -5], [5, 5], [0, 0], 0),
    (A.OBJ_CORNER2, [-2, -2], [2, 2], [0, 0], A.PRED_SUM_LE_1),
    (A.OBJ_NANRIGHT1, [-2], [2], [0], 0),
])
@pytest.mark.parametrize("groups", [1, 3])
def test_trajectory_parity_with_reference(engine, ref, obj, lo, hi, start, pred, groups):
    s = quick(groups=groups, seed=7)
    g = engine.minimize_builtin(obj, lo, hi, s, start, predicate=pred)
    r = ref.minimize_builtin(obj, lo, hi, s, start, predicate=pred)
    assert g.evals == r.evals
    assert len(g.temperature_trace) == len(r.temperature_trace)
    for (tg, fg), (tr, fr) in zip(g.temperature_trace, r.temperature_trace):
        assert tg == tr
        assert abs(fg - fr) <= 1e-12 * max(abs(fr), 1e-12)
    assert np.allclose(g.best_point, r.best_point, rtol=1e-12, atol=1e-14)


def test_static_cost_trajectory_parity(engine, ref, eq_surface):
    """C1 schedule (acceptance.cpp:318-323) on the equity 3m slice: the GPU
    annealer follows the reference trajectory (same evals, same trace)."""
    from oracles import atm_vol_guess

    for seed in (1, 2, 3):
        s = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=32, t_min=1e-7, seed=seed)
        g = engine.calibrate_static_T1(eq_surface, 0, None, s, None, trace=True)
        start = [atm_vol_guess(eq_surface, 0), 1.0, 0.5, -0.3]
        r = ref.minimize_cost(pkg.MODEL_STATIC, eq_surface, 0, [1e-4, 0, 1e-4, -1], [2, 1, 10, 1], s, start)
        assert g.evals == r.evals
        assert len(g.temperature_trace) == len(r.temperature_trace)
        tg = np.array([f for _, f in g.temperature_trace])
        tr = np.array([f for _, f in r.temperature_trace])
        assert np.max(np.abs(tg - tr) / np.abs(tr)) < 1e-10
        assert abs(g.final_cost - r.best_value) <= 1e-10 * r.best_value
        gp = [g.params[k] for k in ("alpha", "beta", "nu", "rho")]
        assert np.allclose(gp, r.best_point, rtol=1e-8, atol=1e-10)
