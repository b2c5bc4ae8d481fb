"""T_II step chain with and without programmatic dependent launch
(SABR_T2_PDL, pdl.cuh), whole-run device time, interleaved: C4 (32 chains,
one 250-step slice, 2 levels) and C5 (2048 chains, 20x30 surface, one SA
step), FP64 and FP32:

    python tools/t2_pdl_ab.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2407_20713_b200 as pkg  # noqa: E402

eng = pkg.Engine(0)
dev = torch.device("cuda:0")
stream = torch.cuda.current_stream(dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for what in ("c4", "c5"):
    for precision in ("fp64", "fp32"):
        if what == "c4":
            surf, fixed, sch, plan = bench.c4_setup(levels=2)
            bounds = None
        else:
            surf, bounds, sch, plan = bench.c5_setup()
            fixed = None
        plan.precision = precision
        best = {}
        for _ in range(4):
            for pdl in ("1", "0"):
                os.environ["SABR_T2_PDL"] = pdl
                torch.cuda.synchronize(dev)
                e0.record(stream)
                rep = eng.calibrate_case2_T2(surf, bounds, sch, plan, fixed)
                e1.record(stream)
                torch.cuda.synchronize(dev)
                t = eng.last_timing()
                secs = e0.elapsed_time(e1) / 1e3
                best.setdefault(pdl, []).append((t.path_steps / secs, rep.final_cost))
        for pdl, r in best.items():
            m = max(r)
            print(f"{what} {precision} pdl={pdl}: {m[0]:.4e} path-steps/s, cost {m[1]:.12e}",
                  flush=True)
eng.close()
