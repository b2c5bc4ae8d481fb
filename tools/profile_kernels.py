"""Small, single-GPU driver for ncu captures of the hot kernels.

  python tools/profile_kernels.py sa      # C2 static level kernel (1e5 chains, 3 levels)
  python tools/profile_kernels.py case1   # C3 Case I level kernel (1e5 chains, 3 levels)
  python tools/profile_kernels.py t2      # C4 T_II: one level, 3 SA steps (MC tile kernel)
  python tools/profile_kernels.py mc      # price_european_batch, 2^20 paths (C4 pricing)
  python tools/profile_kernels.py c5      # C5 T_II: full Case II, 20x30 surface, 512 chains, 1 step
  python tools/profile_kernels.py sa_full     # the whole C2 schedule on slice 0 (412 levels)
  python tools/profile_kernels.py case1_full  # the whole C3 schedule (412 levels, beta = 1)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2407_20713_b200 as pkg  # noqa: E402


def main(mode):
    eng = pkg.Engine(0)
    fx = pkg.parse_surface(os.path.join(ROOT, "tests", "data", "eurusd.csv"))
    eq = pkg.parse_surface(os.path.join(ROOT, "tests", "data", "eurostoxx50.csv"))
    if mode == "sa":
        s = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=12_500, groups=8,
                                  t_min=2.0 * 0.96 ** 2 * 0.999, max_evals=10 ** 12, seed=1)
        r = eng.calibrate_static_T1(fx, 0, None, s, None)
    elif mode == "case1":
        s = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=12_500, groups=8,
                                  t_min=2.0 * 0.96 ** 2 * 0.999, max_evals=10 ** 12, seed=1)
        r = eng.calibrate_dynamic_case1_T1(fx, None, s, {"beta": 1.0})
    elif mode in ("sa_full", "case1_full"):
        s = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=12_500, groups=8,
                                  t_min=1e-7, max_evals=10 ** 12, seed=1)
        if mode == "sa_full":
            r = eng.calibrate_static_T1(fx, 0, None, s, None)
        else:
            r = eng.calibrate_dynamic_case1_T1(fx, None, s, {"beta": 1.0})
    elif mode == "t2":
        surf = pkg.VolSurface(eq.spot, [eq.slices[2]])
        fixed = {"a": 0.0, "b": 0.0, "q_rho": 0.0, "q_nu": 0.0, "d_rho": 0.0, "d_nu": 0.0, "beta": 1.0}
        s = pkg.AnnealingSchedule(t0=2.0, cooling=0.5, chain_length=3, workers=32, t_min=1.5, seed=1)
        plan = pkg.SimulationPlan(num_paths=100_000, seed=1, rng=os.environ.get("SABR_RNG", "xoshiro"),
                                  precision=os.environ.get("SABR_PRECISION", "fp64"))
        r = eng.calibrate_case2_T2(surf, None, s, plan, fixed)
    elif mode == "mc":
        plan = pkg.SimulationPlan(num_paths=1 << 20, seed=3, rng=os.environ.get("SABR_RNG", "xoshiro"),
                                  precision=os.environ.get("SABR_PRECISION", "fp64"))
        p = pkg.StaticSabrParams(0.375162, 0.999999, 0.331441, -0.999999)
        r = eng.price_european_batch(p, 2257.37, [2257.37], 0.018196, 0.034516, 0.495890, plan)
    elif mode == "c5":
        import bench

        surf, bounds, s, plan = bench.c5_setup(chains=512)
        plan.precision = os.environ.get("SABR_PRECISION", "fp64")
        r = eng.calibrate_case2_T2(surf, bounds, s, plan, None)
    else:
        raise SystemExit(__doc__)
    print(mode, "evals" if hasattr(r, "evals") else "", getattr(r, "evals", r))
    t = eng.last_timing()  # MC modes: candidate-path-steps of the run (tools/update_flops.py units)
    print("path_steps", int(t.path_steps), "kernel_launches", int(t.kernel_launches))
    eng.close()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "sa")
