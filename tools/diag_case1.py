"""Dump GPU vs reference Case I costs (diagnostic; run on the GPU box)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2407_20713_b200 as pkg
from oracles import Ref
from test_gpu_costs import case1_vectors, static_vectors
eng, ref = pkg.Engine(0), Ref()
out = {}
for name in ("eurostoxx50", "eurusd"):
    s = pkg.parse_surface(os.path.join(ROOT, "tests/data", name + ".csv"))
    P = case1_vectors(10_000, 43)
    g = eng.cost_batch(pkg.MODEL_CASE1, s, P)
    w = ref.cost_case1(s, P)
    vg = eng.implied_vol_batch(pkg.MODEL_CASE1, s, P)
    out[name] = (P, g, w, vg)
np.savez(os.path.join(ROOT, "gpurun_out/diag_case1.npz"),
         **{f"{k}_{i}": v for k, t in out.items() for i, v in enumerate(t)})
print("ok")
