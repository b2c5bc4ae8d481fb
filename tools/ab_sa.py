"""A/B of two engine builds on the SA level kernels: C2 (static, 1e5 chains,
EUR/USD slice 0) and C3 (Case I, beta = 1, 1e5 chains), level time over the
first levels of the schedule, interleaved:

    python tools/ab_sa.py paper_2407_20713_b200/lib/libsabr_b200.so other.so"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2407_20713_b200 as pkg  # noqa: E402
from paper_2407_20713_b200 import _abi  # noqa: E402

libs = sys.argv[1:]
engs = [pkg.Engine(0, lib=_abi.load_library(p)) for p in libs]
for e in engs:
    e.set_profiling(True)
fx = pkg.parse_surface(os.path.join(ROOT, "tests", "data", "eurusd.csv"))
s = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=12_500, groups=8,
                          t_min=float(os.environ.get("AB_TMIN", 2.0 * 0.96 ** 19 * 0.999)), max_evals=10 ** 12, seed=1)


def run(e, what):
    if what == "c2":
        r = e.calibrate_static_T1(fx, 0, None, s, None)
    else:
        r = e.calibrate_dynamic_case1_T1(fx, None, s, {"beta": 1.0})
    t = e.last_timing()
    return 1e3 * t.kernel_ms / t.kernel_launches, r.final_cost


for what in ("c2", "c3"):
    best = [1e30] * len(engs)
    costs = [None] * len(engs)
    for _ in range(4):
        for i, e in enumerate(engs):
            us, c = run(e, what)
            best[i] = min(best[i], us)
            costs[i] = c
    print(what, " | ".join(f"{os.path.basename(libs[i])}: {best[i]:.1f} us/level (cost {costs[i]:.12e})"
                          for i in range(len(engs))), flush=True)
