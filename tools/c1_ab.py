"""A/B of two engine builds on C1 (calibrate_static_T1, EURO STOXX 50 slice 0,
32 chains, the acceptance schedule): best of six interleaved calls each.

    python tools/c1_ab.py lib_a.so lib_b.so"""
import os, sys, time
sys.path.insert(0, os.getcwd())
import paper_2407_20713_b200 as pkg
from paper_2407_20713_b200 import _abi
libs = sys.argv[1:]
engs = [pkg.Engine(0, lib=_abi.load_library(p)) for p in libs]
eq = pkg.parse_surface('tests/data/eurostoxx50.csv')
s = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=32, t_min=1e-7, seed=1)
best = [1e9] * len(engs)
for _ in range(6):
    for i, e in enumerate(engs):
        e.calibrate_static_T1(eq, 0, None, s)
        t0 = time.perf_counter(); r = e.calibrate_static_T1(eq, 0, None, s); best[i] = min(best[i], time.perf_counter() - t0)
print(" | ".join(f"{os.path.basename(l)}: {b*1e3:.2f} ms" for l, b in zip(libs, best)))
