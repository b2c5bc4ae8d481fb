import os, sys
sys.path.insert(0, os.getcwd())
import bench, paper_2407_20713_b200 as pkg
eng = pkg.Engine(0)
surf, fixed, sch, plan = bench.c4_setup(levels=1)
plan.precision = os.environ.get("P", "fp32")
sch = pkg.AnnealingSchedule(t0=sch.t0, cooling=sch.cooling, chain_length=4, workers=sch.workers, t_min=sch.t0*0.999, seed=1)
eng.calibrate_case2_T2(surf, None, sch, plan, fixed)
