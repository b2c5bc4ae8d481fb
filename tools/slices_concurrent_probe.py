"""C2's four EUR/USD slice calibrations run one after another (the bench's
step) and concurrently (one engine context and stream per slice, one host
thread each), to measure what co-resident level kernels of independent
slices buy: a single slice's level grid (1042 one-warp CTAs) holds 7 warps
per SM, the register file 10.

    python tools/slices_concurrent_probe.py [levels [engine .so ...]]"""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2407_20713_b200 as pkg  # noqa: E402
from paper_2407_20713_b200 import _abi  # noqa: E402

levels = int(sys.argv[1]) if len(sys.argv) > 1 else 60
libs = sys.argv[2:] or [None]
fx = pkg.parse_surface(os.path.join(ROOT, "tests", "data", "eurusd.csv"))
n_sl = len(fx.slices)
sch = bench.c2_schedule(1, max_evals=bench.C2_CHAINS_PER_GPU * 100 * levels + 1)


def seq():
    reps = [engs[0].calibrate_static_T1(fx, s, None, sch, None) for s in range(n_sl)]
    torch.cuda.synchronize()
    return reps


def conc():
    reps = [None] * n_sl

    def run(s):
        reps[s] = engs[s].calibrate_static_T1(fx, s, None, sch, None)

    th = [threading.Thread(target=run, args=(s,)) for s in range(n_sl)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    return reps


for lib in libs:
    engs = [pkg.Engine(0, lib=_abi.load_library(lib) if lib else None) for _ in range(n_sl)]
    for name, f in (("sequential", seq), ("concurrent", conc), ("slices API", lambda: engs[0].calibrate_static_T1_slices(
            fx, None, None, sch, None))):
        f()
        best = None
        for _ in range(3):
            t0 = time.perf_counter()
            reps = f()
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        evals = sum(r.evals - 1 for r in reps)
        print(f"{os.path.basename(lib or 'default')} {name}: {best * 1e3:.1f} ms, {evals / best:.4e} cost-evals/s, "
              f"costs {[f'{r.final_cost:.6e}' for r in reps]}", flush=True)
    for e in engs:
        e.close()
