"""The T_I level kernel variants must produce bit-identical annealer
trajectories: three chains per thread (the static default), two (the Case I
default), one chain per thread in the same kernel (SABR_SA_CPT=1) and the
general one-chain kernel (SABR_SA_CPT=0);
the FAST propose/exp path (one reflection, unsaturated exp; kernels_sa.cu
propose_coord_fast) vs the general one (SABR_SA_FAST=0).  The factored slice
cost (slice_qr.hpp, default) and the per-quote sum (SABR_SA_COST=quotes)
round differently, so between them the decisions (evals, trace length) must
agree and the values to 1e-12.  The switches are read once per process, so
each variant runs in its own subprocess."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import paper_2407_20713_b200 as pkg
eng = pkg.Engine(0)
eq = pkg.parse_surface("tests/data/eurostoxx50.csv")
fx = pkg.parse_surface("tests/data/eurusd.csv")
out = {}
# odd chain count: the last thread of the multi-chain kernel has an inactive chain
s = pkg.AnnealingSchedule(t0=2.0, cooling=0.9, chain_length=60, workers=301, groups=3, t_min=1e-4, seed=5)
r = eng.calibrate_static_T1(eq, 1, None, s, None, trace=True)
out["static"] = [r.final_cost.hex(), {k: v.hex() for k, v in r.params.items()}, r.evals,
                 [f.hex() for _, f in r.temperature_trace]]
r = eng.calibrate_static_T1(fx, 2, None, s, {"beta": 0.5}, trace=True)
out["static_fixed"] = [r.final_cost.hex(), {k: v.hex() for k, v in r.params.items()}, r.evals,
                       [f.hex() for _, f in r.temperature_trace]]
# eval cap reached inside a level
s2 = pkg.AnnealingSchedule(t0=2.0, cooling=0.8, chain_length=50, workers=77, t_min=1e-2, seed=9, max_evals=20000)
r = eng.calibrate_static_T1(fx, 0, None, s2, None, trace=True)
out["static_cap"] = [r.final_cost.hex(), r.evals, [f.hex() for _, f in r.temperature_trace]]
s3 = pkg.AnnealingSchedule(t0=2.0, cooling=0.8, chain_length=40, workers=129, t_min=1e-3, seed=2)
r = eng.calibrate_dynamic_case1_T1(fx, None, s3, None, trace=True)
out["case1"] = [r.final_cost.hex(), {k: v.hex() for k, v in r.params.items()}, r.evals,
                [f.hex() for _, f in r.temperature_trace]]
# beta not searched: the two-chain kernel takes f^(1-beta) per CTA, the others per chain
r = eng.calibrate_dynamic_case1_T1(eq, None, s3, {"beta": 0.7}, trace=True)
out["case1_beta_fixed"] = [r.final_cost.hex(), {k: v.hex() for k, v in r.params.items()}, r.evals,
                           [f.hex() for _, f in r.temperature_trace]]
# one-CTA runs (<= 64 chains): every level in one launch unless SABR_SA_PERSIST=0
s4 = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=32, t_min=1e-7, seed=2)
r = eng.calibrate_static_T1(eq, 1, None, s4, None, trace=True)
out["small_static"] = [r.final_cost.hex(), {k: v.hex() for k, v in r.params.items()}, r.evals,
                       [f.hex() for _, f in r.temperature_trace]]
s5 = pkg.AnnealingSchedule(t0=2.0, cooling=0.9, chain_length=50, workers=21, groups=3, t_min=1e-5, seed=7,
                           max_evals=150000)
r = eng.calibrate_dynamic_case1_T1(fx, None, s5, {"beta": 1.0}, trace=True)
out["small_case1_cap"] = [r.final_cost.hex(), {k: v.hex() for k, v in r.params.items()}, r.evals,
                          [f.hex() for _, f in r.temperature_trace]]
print(json.dumps(out))
"""


def run_variant(cpt, fast=None, cost=None, persist=None):
    env = dict(os.environ)
    for k in ("SABR_SA_CPT", "SABR_SA_FAST", "SABR_SA_COST", "SABR_SA_PERSIST"):
        env.pop(k, None)
    if persist is not None:
        env["SABR_SA_PERSIST"] = str(persist)
    if cpt is not None:
        env["SABR_SA_CPT"] = str(cpt)
    if fast is not None:
        env["SABR_SA_FAST"] = str(fast)
    if cost is not None:
        env["SABR_SA_COST"] = cost
    p = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("cost", [None, "quotes"])
def test_multi_chain_kernel_matches_single_chain_kernels(cost):
    multi = run_variant(None, cost=cost)
    for cpt in ((1, 0, 2, 3) if cost is None else (0,)):
        single = run_variant(cpt, cost=cost)
        assert multi.keys() == single.keys()
        for k in multi:
            assert multi[k] == single[k], (cpt, k)


def _close(a, b, rel):
    a, b = float.fromhex(a), float.fromhex(b)
    return abs(a - b) <= rel * max(abs(a), abs(b), 1e-300)


def test_factored_cost_matches_per_quote_cost():
    qr = run_variant(None)
    quotes = run_variant(None, cost="quotes")
    for k in qr:
        a, b = qr[k], quotes[k]
        assert _close(a[0], b[0], 1e-12), k
        tr_a, tr_b = a[-1], b[-1]
        assert len(tr_a) == len(tr_b), k
        assert all(_close(x, y, 1e-12) for x, y in zip(tr_a, tr_b)), k
        if isinstance(a[1], dict):
            assert a[2] == b[2], k  # evals
            assert all(_close(a[1][p], b[1][p], 1e-9) for p in a[1]), k
        else:
            assert a[1] == b[1], k


def test_fast_propose_matches_general_propose():
    fast = run_variant(None)
    general = run_variant(None, fast=0)
    for k in fast:
        assert fast[k] == general[k], k


def test_one_launch_run_matches_per_level_launches():
    """sa_run_small_kernel (all levels of a one-CTA run in one launch, with an
    eval cap reached inside a level) against the per-level kernels."""
    persistent = run_variant(None)
    per_level = run_variant(None, persist=0)
    for k in persistent:
        assert persistent[k] == per_level[k], k
