"""One rank of tests/test_gpu_multirank_engine.py: the engine's rank
decomposition (chains split over ranks, per-level record all-gather, merge
kernel) with the exchange over a gloo process group on the host.  Ranks may
share one GPU.  Prints the reports of every workload as hex JSON (rank 0).

  python tests/mr_engine_worker.py RANK WORLD PORT [peer]

With "peer" the T_I calibrators exchange their level records through the
fused peer-memory path (sabr_ctx_enable_peer_exchange: CUDA IPC mailboxes,
here between processes on one GPU) instead of the host all-gather.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2407_20713_b200 as pkg  # noqa: E402


def report_key(r):
    return [r.final_cost.hex(), {k: v.hex() for k, v in sorted(r.params.items())}, r.evals,
            [f.hex() for _, f in r.temperature_trace], [row.model.hex() for row in r.rows]]


def workloads(eng):
    data = os.path.join(ROOT, "tests", "data")
    fx = pkg.parse_surface(os.path.join(data, "eurusd.csv"))
    eq = pkg.parse_surface(os.path.join(data, "eurostoxx50.csv"))
    out = {}
    s = pkg.AnnealingSchedule(t0=2.0, cooling=0.85, chain_length=40, workers=301, groups=3, t_min=1e-4, seed=7)
    out["static"] = report_key(eng.calibrate_static_T1(fx, 1, None, s, None, trace=True))
    # every slice in one call: side by side on child streams (one rank, or
    # ranks on peer mailboxes: each child its own), else one after another
    for i, r in enumerate(eng.calibrate_static_T1_slices(fx, [3, 1, 0], None, s, None, trace=True)):
        out[f"static_slices_{i}"] = report_key(r)
    cap = pkg.AnnealingSchedule(t0=2.0, cooling=0.8, chain_length=50, workers=77, groups=2, t_min=1e-2, seed=9,
                                max_evals=20000)
    out["static_cap"] = report_key(eng.calibrate_static_T1(eq, 0, None, cap, {"beta": 0.9}, trace=True))
    s1 = pkg.AnnealingSchedule(t0=2.0, cooling=0.7, chain_length=20, workers=129, groups=2, t_min=1e-3, seed=2)
    out["case1"] = report_key(eng.calibrate_dynamic_case1_T1(fx, None, s1, None, trace=True))
    surf = pkg.VolSurface(eq.spot, [eq.slices[2]])
    fixed = {"a": 0.0, "b": 0.0, "q_rho": 0.0, "q_nu": 0.0, "d_rho": 0.0, "d_nu": 0.0, "beta": 1.0}
    s2 = pkg.AnnealingSchedule(t0=2.0, cooling=0.5, chain_length=3, workers=5, groups=2, t_min=0.2, seed=3)
    out["case2_T2"] = report_key(eng.calibrate_case2_T2(surf, None, s2, pkg.SimulationPlan(num_paths=4096, seed=1),
                                                        fixed, trace=True))
    # fewer chains than ranks (1 chain): path tiles split over the ranks, partials all-gathered per step
    s4 = pkg.AnnealingSchedule(t0=2.0, cooling=0.5, chain_length=4, workers=1, groups=1, t_min=0.2, seed=4)
    out["case2_T2_one_chain"] = report_key(eng.calibrate_case2_T2(surf, None, s4, pkg.SimulationPlan(
        num_paths=20000, seed=2), fixed, trace=True))
    # the path split forced with more chains than ranks (SABR_T2_SHARD=paths), reference streams
    os.environ["SABR_T2_SHARD"] = "paths"
    out["case2_T2_paths"] = report_key(eng.calibrate_case2_T2(surf, None, s2, pkg.SimulationPlan(
        num_paths=10000, seed=1, block_size=1000), fixed, trace=True))
    del os.environ["SABR_T2_SHARD"]
    s3 = pkg.AnnealingSchedule(t0=2.0, cooling=0.5, chain_length=4, workers=6, groups=2, t_min=0.1, seed=2)
    out["case2_formula"] = report_key(eng.calibrate_case2_formula(fx, None, s3, {"beta": 1.0}, trace=True))
    return out


def main():
    rank, world, port = (int(x) for x in sys.argv[1:4])
    peer = len(sys.argv) > 4 and sys.argv[4] == "peer"
    eng = pkg.Engine(0)
    if world > 1:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)

        def allgather(send: bytes) -> bytes:
            t = torch.frombuffer(bytearray(send), dtype=torch.uint8)
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(parts, t)
            return b"".join(bytes(p.numpy().tobytes()) for p in parts)

        eng.init_host_exchange(rank, world, allgather)
        if peer:
            eng.enable_peer_exchange()
    out = workloads(eng)
    eng.close()
    if world > 1:
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out))


if __name__ == "__main__":
    main()
