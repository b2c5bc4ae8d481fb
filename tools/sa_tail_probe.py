import os, sys
sys.path.insert(0, os.getcwd())
import paper_2407_20713_b200 as pkg
eng = pkg.Engine(0); eng.set_profiling(True)
fx = pkg.parse_surface("tests/data/eurusd.csv")
for L in (1, 2, 10, 100):
    s = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=L, workers=100000, groups=1,
                              t_min=2.0 * 0.96 ** 49 * 0.999, max_evals=10 ** 12, seed=1)
    eng.calibrate_static_T1(fx, 0, None, s, None)
    r = eng.calibrate_static_T1(fx, 0, None, s, None)
    t = eng.last_timing()
    print(f"L={L:4d} level kernel {1e3 * t.kernel_ms / t.kernel_launches:8.2f} us  launches {t.kernel_launches}", flush=True)
eng.close()
