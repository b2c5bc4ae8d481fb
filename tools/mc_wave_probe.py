"""MC tile-kernel throughput vs path count at the C4 shape (32 candidates,
one T = 1 slice, 250 steps): how much the partial last wave of blocks costs.
  python tools/mc_wave_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2407_20713_b200 as pkg  # noqa: E402

eng = pkg.Engine(0)
eng.set_profiling(True)
for paths in (75_776, 100_000, 113_664, 151_552, 227_328):
    surf, fixed, sch, plan = bench.c4_setup(levels=2)
    plan.num_paths = paths
    small = pkg.AnnealingSchedule(t0=2.0, cooling=0.5, chain_length=2, workers=32, t_min=1.5, seed=1)
    eng.calibrate_case2_T2(surf, None, small, plan, fixed)
    rep = eng.calibrate_case2_T2(surf, None, sch, plan, fixed)
    t = eng.last_timing()
    blocks = -(-paths // 512) * 4
    print(f"paths {paths:7d}: blocks {blocks:5d} ({blocks / 592:.2f} waves), kernel "
          f"{t.path_steps / (t.kernel_ms / 1e3):.3e} path-steps/s")
