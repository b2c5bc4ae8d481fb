"""C3 (Case I, EUR/USD, beta = 1, 1e5 chains) level-kernel time for A/B runs
of the level-kernel variants (SABR_SA_CPT, SABR_SA_PIPE):

    SABR_SA_CPT=1 python tools/c3_probe.py

prints the device time per level and the cost-evals/s over the first
`levels` levels of the C3 schedule."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2407_20713_b200 as pkg  # noqa: E402

levels = int(sys.argv[1]) if len(sys.argv) > 1 else 20
eng = pkg.Engine(0)
eng.set_profiling(True)
fx = pkg.parse_surface(os.path.join(ROOT, "tests", "data", "eurusd.csv"))
s = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=12_500, groups=8,
                          t_min=2.0 * 0.96 ** (levels - 1) * 0.999, max_evals=10 ** 12, seed=1)
for _ in range(2):
    r = eng.calibrate_dynamic_case1_T1(fx, None, s, {"beta": 1.0})
t = eng.last_timing()
us = 1e3 * t.kernel_ms / t.kernel_launches
print(f"cpt {os.environ.get('SABR_SA_CPT', 'default')} pipe {os.environ.get('SABR_SA_PIPE', '0')}: "
      f"{t.kernel_launches} levels, {us:.1f} us per level, {1e7 / us * 1e6:.3e} evals/s, "
      f"final cost {r.final_cost:.6e}", flush=True)
eng.close()
