"""Level-kernel time vs chains per GPU (C2 schedule, EUR/USD slice 0): shows
whether the SA level kernel is bound by per-warp latency (time flat in the
warp count) or by issue/pipe throughput (time proportional)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2407_20713_b200 as pkg  # noqa: E402

eng = pkg.Engine(0)
eng.set_profiling(True)
fx = pkg.parse_surface(os.path.join(ROOT, "tests", "data", "eurusd.csv"))
for chains in (148 * 64, 2 * 148 * 64, 4 * 148 * 64, 8 * 148 * 64, 100_000, 12 * 148 * 64, 16 * 148 * 64):
    s = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=chains, groups=1,
                              t_min=2.0 * 0.96 ** 9 * 0.999, max_evals=10 ** 12, seed=1)
    eng.calibrate_static_T1(fx, 0, None, s, None)
    eng.calibrate_static_T1(fx, 0, None, s, None)
    t = eng.last_timing()
    us = 1e3 * t.kernel_ms / t.kernel_launches
    warps = chains / 64
    print(f"chains {chains:7d}  warps/SMSP {warps / 592:5.2f}  level {us:7.1f} us  "
          f"cycles/step/warp {us * 1.965e3 / 100:7.0f}  evals/s {chains * 100 / us * 1e6:.3e}", flush=True)
eng.close()
