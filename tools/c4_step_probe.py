"""One C4 SA level of 4 steps (32 chains, one 250-step slice, 1e5 paths) for
a per-kernel launch list of the T_II step chain:

    ncu --metrics gpu__time_duration.sum --clock-control none --csv \\
        --log-file gpurun_out/c4_launches.csv python tools/c4_step_probe.py
    P=fp64 ... (default fp32)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2407_20713_b200 as pkg  # noqa: E402

eng = pkg.Engine(0)
surf, fixed, sch, plan = bench.c4_setup(levels=1)
plan.precision = os.environ.get("P", "fp32")
sch = pkg.AnnealingSchedule(t0=sch.t0, cooling=sch.cooling, chain_length=4, workers=sch.workers,
                            t_min=sch.t0 * 0.999, seed=1)
eng.calibrate_case2_T2(surf, None, sch, plan, fixed)
eng.close()
