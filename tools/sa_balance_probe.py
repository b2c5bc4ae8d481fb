"""Level-kernel time at chain counts that load every SM sub-partition (SMSP)
equally: n = k * 592 * 32 chains puts k lane-chains on every scheduler
(k / C warps of C chains per thread).  Run once per SABR_SA_CPT (1, 2, 3):

    SABR_SA_CPT=3 python tools/sa_balance_probe.py 3 6

prints, per k, the level time and the cost per lane-chain-step, i.e. how the
scheduler's throughput depends on the number of resident chain streams.  With
it, the time of a perfectly balanced 1e5-chain level (5.28 lane-chains per
scheduler) can be read off without building it."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2407_20713_b200 as pkg  # noqa: E402

eng = pkg.Engine(0)
eng.set_profiling(True)
fx = pkg.parse_surface(os.path.join(ROOT, "tests", "data", "eurusd.csv"))
cpt = os.environ.get("SABR_SA_CPT", "3")
ks = [int(k) for k in sys.argv[1:]] or [1, 2, 3, 4, 5, 6]
for k in ks + [0]:
    chains = k * 592 * 32 if k else 100_000
    s = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=chains, groups=1,
                              t_min=2.0 * 0.96 ** 9 * 0.999, max_evals=10 ** 12, seed=1)
    eng.calibrate_static_T1(fx, 0, None, s, None)
    eng.calibrate_static_T1(fx, 0, None, s, None)
    t = eng.last_timing()
    us = 1e3 * t.kernel_ms / t.kernel_launches
    lc = chains / (592 * 32)
    print(f"cpt {cpt} lane-chains/SMSP {lc:5.2f} chains {chains:7d} level {us:7.1f} us  "
          f"cycles per lane-chain-step {us * 1.965e3 / 100 / lc:6.1f}  evals/s {chains * 100 / us * 1e6:.3e}",
          flush=True)
eng.close()
