"""A/B of two engine builds on the MC calibration items (C4 and C5 FP64/FP32,
path-steps/s of the MC kernels and of the whole run), interleaved so clock
drift affects both alike:

    python tools/ab_mc.py paper_2407_20713_b200/lib/libsabr_b200.so other.so"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2407_20713_b200 as pkg  # noqa: E402
from paper_2407_20713_b200 import _abi  # noqa: E402


def run(eng, what, precision):
    if what == "c4":
        surf, fixed, sch, plan = bench.c4_setup(levels=2)
        bounds = None
    else:
        surf, bounds, sch, plan = bench.c5_setup()
        fixed = None
    plan.precision = precision
    eng.calibrate_case2_T2(surf, bounds, sch, plan, fixed)
    eng.calibrate_case2_T2(surf, bounds, sch, plan, fixed)
    t = eng.last_timing()
    return t.path_steps / (t.kernel_ms / 1e3), t.path_steps / (t.total_ms / 1e3)


libs = sys.argv[1:]
engs = [pkg.Engine(0, lib=_abi.load_library(p)) for p in libs]
for e in engs:
    e.set_profiling(True)
for what in ("c4", "c5"):
    for precision in ("fp64", "fp32"):
        vals = [[] for _ in engs]
        for _ in range(3):
            for i, e in enumerate(engs):
                vals[i].append(run(e, what, precision))
        print(what, precision, " | ".join(f"{os.path.basename(libs[i])}: kernel {max(k for k, _ in v):.4e} "
                                          f"run {max(w for _, w in v):.4e}" for i, v in enumerate(vals)), flush=True)
