import time, sys
sys.path.insert(0, '/root/repo')
import paper_2407_20713_b200 as pkg
eng = pkg.Engine(0)
eq = pkg.parse_surface('/root/repo/tests/data/eurostoxx50.csv')
for L in (100, 50, 10, 1):
    s = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=L, workers=32, t_min=1e-7, seed=2)
    eng.calibrate_static_T1(eq, 1, None, s)
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); r = eng.calibrate_static_T1(eq, 1, None, s); ts.append(time.perf_counter() - t0)
    print(f"L={L}: {min(ts)*1e3:.2f} ms, evals {r.evals}, per level {min(ts)/412*1e6:.1f} us")
