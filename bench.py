#!/usr/bin/env python
"""Benchmark of the B200 SABR calibration engine ("Measurement").

Headline workload (BASELINE.json configs[1], "C2"): static SABR with the
Hagan/Obloj formula (Eq. 7), parallel SA calibration of every maturity of the
EUR/USD surface (proj/data/eurusd.csv) with 1e5 chains per GPU.  One step =
calibrate_static_T1 on each of the 4 slices (t0=2, cooling 0.96, L=100,
t_min=1e-7 -> 412 temperature levels, 4.1e9 cost-evals per slice per 1e5
chains).  Metric: SA cost-evals/s (whole job).  Secondary line items: the
Monte Carlo objective (C4: calibrate_case2_T2 on the T=1 equity slice, 1e5
paths x 250 steps per cost eval) as path-steps/s, and Case I (C3).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Under torchrun each rank drives one GPU; chains are split over ranks (weak
scaling: 1e5 chains per GPU) and the per-level record exchange is NCCL.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

C2_CHAINS_PER_GPU = 100_000
C2_WORKERS, C2_GROUPS = 12_500, 8
LEVELS_C1 = 412  # (2 * 0.96^k >= 1e-7)


def c2_schedule(n_gpus, seed=1, max_evals=None):
    import paper_2407_20713_b200 as pkg

    n = C2_CHAINS_PER_GPU * n_gpus
    return pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=C2_WORKERS * n_gpus,
                                 groups=C2_GROUPS, t_min=1e-7,
                                 max_evals=max_evals or (n * 100 * LEVELS_C1 + 1), seed=seed)


def c4_setup(levels=2):
    """C4: calibrate_case2_T2 on the T=1 equity slice, dynamics pinned static."""
    import paper_2407_20713_b200 as pkg

    eq = pkg.parse_surface(os.path.join(ROOT, "tests", "data", "eurostoxx50.csv"))
    surf = pkg.VolSurface(eq.spot, [eq.slices[2]])
    fixed = {"a": 0.0, "b": 0.0, "q_rho": 0.0, "q_nu": 0.0, "d_rho": 0.0, "d_nu": 0.0, "beta": 1.0}
    t_min = 2.0 * 0.96 ** (levels - 1) * 0.999
    sch = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=32, t_min=t_min, seed=1,
                                max_evals=10 ** 12)
    plan = pkg.SimulationPlan(num_paths=100_000, dt=1 / 250, seed=1, rng="xoshiro")
    return surf, fixed, sch, plan


# C5 (BASELINE.json configs[4]): full Case II MC calibration on the synthetic
# 20-maturity x 30-strike surface (tests/data/synth20x30.csv, generated from
# the published FX Case II fit by tests/golden/make_synth.py).  Search box:
# the default Case II box narrowed to +-2% of its width around that fit (the
# full box at T = t0 proposes exploding dynamics, which the reference aborts
# on), every parameter free.
CASE2_DEFAULTS = [("alpha", 1e-4, 2.0), ("beta", 0.0, 1.0), ("rho0", -1.0, 1.0), ("q_rho", -15.0, 15.0),
                  ("d_rho", -1.0, 1.0), ("nu0", 1e-4, 10.0), ("q_nu", -15.0, 15.0), ("d_nu", -1.0, 1.0),
                  ("a", 0.0, 150.0), ("b", 0.0, 150.0)]
FX_CASE2 = [0.154037, 1.0, -0.693682, 0.345973, -0.200342, 7.541424, -0.992551, 0.339807, 0.0, 150.0]


def c5_bounds(width=0.02):
    out = {}
    for (name, lo, hi), p in zip(CASE2_DEFAULTS, FX_CASE2):
        h = width * (hi - lo)
        out[name] = (max(lo, p - h), min(hi, p + h))
    return out


def c5_setup(chains=2048, num_paths=4096):
    """C5 sample: one temperature level, one SA step of `chains` chains."""
    import paper_2407_20713_b200 as pkg

    surf = pkg.parse_surface(os.path.join(ROOT, "tests", "data", "synth20x30.csv"))
    sch = pkg.AnnealingSchedule(t0=2.0, cooling=0.5, chain_length=1, workers=chains // 8, groups=8, t_min=1.5,
                                seed=1, max_evals=10 ** 12)
    plan = pkg.SimulationPlan(num_paths=num_paths, dt=1 / 250, seed=1, rng="xoshiro")
    return surf, c5_bounds(), sch, plan


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for name, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def flush_l2(torch, dev):
    buf = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    buf.zero_()
    del buf


def surface_bytes(surface):
    ns, nq = len(surface.slices), surface.total_quotes()
    return 8 * (4 * nq + 3 * ns) + 4 * (ns + 1)


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2407_20713_b200 as pkg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SABR_BENCH_SHARED_GPU=1 (testing only): every rank on cuda:0, gloo for torch's collectives
    # and the host all-gather as the engine transport, so the multi-rank code of this script runs
    # on a single-GPU box; the numbers are not a scaling measurement
    shared = os.environ.get("SABR_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream(dev)
    eng = pkg.Engine(local, stream=stream.cuda_stream)
    if world > 1 and shared:
        def allgather_gloo(send: bytes) -> bytes:
            t = torch.frombuffer(bytearray(send), dtype=torch.uint8)
            parts = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(parts, t)
            return b"".join(bytes(p.numpy().tobytes()) for p in parts)

        eng.init_host_exchange(rank, world, allgather_gloo)
        ok = torch.tensor([1], dtype=torch.int32)
        try:
            eng.enable_peer_exchange()
        except pkg.SabrError:
            ok.fill_(0)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok) == 1:
            transport = "fused peer-memory exchange (shared-GPU test mode)"
        else:
            eng.disable_peer_exchange()
            transport = "host all-gather (shared-GPU test mode)"
    elif world > 1:
        uid = torch.zeros(129, dtype=torch.uint8, device=dev)  # NCCL unique id + "ok" byte
        if rank == 0:
            try:
                uid[:128].copy_(torch.frombuffer(bytearray(pkg.Engine.comm_unique_id()), dtype=torch.uint8))
                uid[128] = 1
            except pkg.SabrError:
                pass
        dist.broadcast(uid, 0)
        ok = torch.tensor([0], dtype=torch.int32, device=dev)
        try:
            if int(uid[128]) != 1:
                raise pkg.SabrError("no NCCL unique id on rank 0")
            eng.init_comm(bytes(uid[:128].cpu().numpy().tobytes()), rank, world)
            ok.fill_(1)
        except pkg.SabrError as e:
            print(f"rank {rank}: engine NCCL init failed ({e})", file=sys.stderr)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok) == 1:
            transport = "NCCL all-gather (engine communicator)"
        else:  # engine cannot open its own communicator: the records go through torch's NCCL group
            def allgather(send: bytes) -> bytes:
                t = torch.frombuffer(bytearray(send), dtype=torch.uint8).to(dev)
                out = torch.empty(world * t.numel(), dtype=torch.uint8, device=dev)
                dist.all_gather_into_tensor(out, t)
                return bytes(out.cpu().numpy().tobytes())

            eng.init_host_exchange(rank, world, allgather)
            transport = "torch.distributed all-gather (host exchange)"
        # fused peer-memory exchange of the level records (CUDA IPC mailboxes over NVLink /
        # NVSwitch, merged inside the level kernel): used when every rank can map the others
        ok = torch.tensor([1], dtype=torch.int32, device=dev)
        try:
            eng.enable_peer_exchange()
        except pkg.SabrError as e:
            print(f"rank {rank}: peer exchange unavailable ({e})", file=sys.stderr)
            ok.fill_(0)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok) == 1:
            transport = "fused peer-memory exchange in the level kernel (CUDA IPC mailboxes)"
        else:
            eng.disable_peer_exchange()
    else:
        transport = "none (1 rank)"
    print(f"bench rank {rank}/{world}: device cuda:{local}, transport: {transport}", file=sys.stderr, flush=True)
    eng.set_profiling(True)

    fx = pkg.parse_surface(os.path.join(ROOT, "tests", "data", "eurusd.csv"))
    sch = c2_schedule(world)

    def step():
        """One step: calibrate every EUR/USD slice (C2), in one call: on one
        rank the four slices' annealers run side by side on their own streams
        (Engine.calibrate_static_T1_slices; with N ranks one after another)."""
        t0 = time.perf_counter()
        reps = eng.calibrate_static_T1_slices(fx, None, None, sch, None)
        wall = time.perf_counter() - t0
        t = eng.last_timing()
        evals = sum(rep.evals - 1 for rep in reps)
        launches = t.total_launches + 3 * len(reps)  # + start, vol and surface-upload kernels per slice
        return evals, launches, t.kernel_ms, t.kernel_launches, wall, reps

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    ev_times, walls, evals_tot, launches_tot, kms_tot, klaunch_tot = [], [], 0, 0, 0.0, 0
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush_l2(torch, dev)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize(dev)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            evals, launches, kms, kl, wall, reps = step()
            e1.record(stream)
            torch.cuda.synchronize(dev)
            ev_times.append(e0.elapsed_time(e1) / 1e3)
            walls.append(wall)
            evals_tot += evals
            launches_tot += launches
            kms_tot += kms
            klaunch_tot += kl
    t_dev = sum(ev_times)
    t_wall = sum(walls)
    if world > 1:
        tt = torch.tensor([t_dev, t_wall], dtype=torch.float64, device="cpu" if shared else dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_dev, t_wall = tt.tolist()
    # evals reported by calibrate_* are global (all ranks' chains)
    value = evals_tot / t_dev
    e2e = evals_tot / t_wall

    # ---- roofline of the dominant kernel (the SA level kernel) ----
    peak = float(np.median([fp64_peak(eng) for _ in range(3)]))
    per_eval = fp64_flops_per_eval()
    # per-launch time = device time of the timed steps / level launches: the
    # sampled per-launch events overlap under programmatic dependent launch
    # (their sum exceeded the step time by ~3%), so the step time bounds it
    avg_launch_s = t_dev / klaunch_tot
    evals_per_launch = evals_tot / klaunch_tot / world  # this rank's chains
    achieved = evals_per_launch * per_eval["flops"] / avg_launch_s / 1e12
    traffic = per_eval.get("dram_bytes_per_launch")
    # the same kernel as FP64-pipe occupancy: every FP64-pipe instruction (DFMA,
    # DADD, DMUL, DSETP, ...) per eval against the lane-instruction peak
    # (= the DFMA FLOP peak / 2), i.e. ncu's sm__pipe_fp64_cycles_active view
    pipe = None
    if per_eval.get("pipe_instr"):
        pa = evals_per_launch * per_eval["pipe_instr"] / avg_launch_s / 1e12
        pipe = {"instr_per_eval": per_eval["pipe_instr"], "achieved_Tinstr_per_s": pa,
                "peak_Tinstr_per_s": peak / 2, "frac": pa / (peak / 2)}

    # and as issue-slot occupancy: warp instructions per eval (ncu) against one
    # instruction per cycle per scheduler (148 SMs x 4) at the sampled SM clock
    issue = None
    clk = clocks.summary().get("sm_mhz") if hasattr(clocks, "summary") else None
    if per_eval.get("warp_instr") and clk:
        ia = evals_per_launch * per_eval["warp_instr"] / avg_launch_s
        ip = 148 * 4 * clk * 1e6
        issue = {"warp_instr_per_eval": per_eval["warp_instr"], "achieved_warp_instr_per_s": ia,
                 "peak_warp_instr_per_s": ip, "frac": ia / ip}

    sec = {}
    if rank == 0 and world == 1 and not args.no_secondary:
        mufu = float(np.median([mufu_peak(eng) for _ in range(3)]))
        sec = secondary(eng, torch, dev, stream, {"fp64_tflops": peak, "mufu_tops": mufu})
        if args.full_configs:
            sec.update(full_configs(eng, torch, dev, stream, {"fp64_tflops": peak, "mufu_tops": mufu}))

    line = {
        "metric": "SA cost-evals/s, static Hagan/Obloj (Eq. 7) calibration, EUR/USD surface, 1e5 chains/GPU",
        "value": value,
        "unit": "cost-evals/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * t_dev / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "reference fixture proj/data/eurusd.csv (4 maturities x 19 strikes), copied to tests/data",
        "config": {"workload": "C2: calibrate_static_T1 on each EUR/USD slice, 1e5 SA chains per GPU "
                               f"(workers {C2_WORKERS}x{world}, groups {C2_GROUPS}), t0=2 cooling=0.96 "
                               "L=100 t_min=1e-7 (412 levels)",
                   "chains": C2_CHAINS_PER_GPU * world, "levels": LEVELS_C1,
                   "cost_evals_per_step": evals_tot / args.steps,
                   "calibration_wall_s": t_wall / (args.steps * len(fx.slices)),
                   "l2": "flushed (256 MB write) before every timed step",
                   "parallelism": f"chains sharded over {world} GPU(s), one 240-byte record all-gather per level; "
                                  + ("the 4 slices' calibrations side by side on 4 streams "
                                     "(calibrate_static_T1_slices)" if world == 1 or transport.startswith("fused")
                                     else "slices one after another (per-level transport all-gather)"),
                   "transport": transport},
        "e2e": {"value": e2e, "unit": "cost-evals/s",
                "h2d_bytes_per_step": len(fx.slices) * (surface_bytes(pkg.VolSurface(fx.spot, [fx.slices[0]])) + 4 * 8 + 400),
                "d2h_bytes_per_step": len(fx.slices) * (400 + 8 * LEVELS_C1 + 8 * 19 + 8 * 5)},
        "gpu_launches": int(launches_tot),
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "kernel": "sa_level_multi_kernel<OBJ_STATIC,4,ALLFREE,QR,3> (3 chains per thread, factored slice cost)",
                     "avg_launch_ms": avg_launch_s * 1e3, "launches": klaunch_tot,
                     "avg_launch_source": "device time of the timed steps / level-kernel launches (one rank: the "
                                          "four slices' level kernels run concurrently, so this is the step's "
                                          "time per launch, not one launch's duration; it includes the "
                                          "start/report kernels and launch gaps)",
                     "flops_per_eval": per_eval["flops"], "flops_source": per_eval["source"],
                     "peak_source": "measured in bench.py (sabr_bench_fp64_peak, DFMA microbenchmark); "
                                    "MEASURED_PEAKS.json has no FP64 figure",
                     "fp64_pipe": pipe,
                     "issue": issue,
                     # SURVEY 8(d)'s per-quote form (4-quote-independent terms hoisted,
                     # 2 divisions per quote): ~1180 FP64 instructions per C2 eval; the
                     # factored slice cost (slice_qr.hpp) executes fp64_instr_per_eval
                     "survey_8d_fp64_instr_per_eval": 1180,
                     "fp64_instr_per_eval": per_eval.get("instr")},
        "clocks": clocks.summary(),
    }
    if sec:
        line["secondary"] = sec
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(fx)
        c1 = line.get("secondary", {}).get("c1_static_calibration")
        m = line["cpu_baseline"].get("matrix")
        if c1 and m:
            # C1 is the one config whose whole reference run is short: same-config wall-time ratio
            ref_s = m[f"threads_{line['cpu_baseline']['cores']}"]["c1_static_calibration_s"]
            c1["reference_s_all_threads"] = ref_s
            c1["speedup_vs_reference_same_config"] = ref_s / c1["value"]
    if world > 1:
        dist.barrier()
    if rank == 0:
        print(json.dumps(line), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


def mufu_peak(eng):
    import ctypes as C

    v = C.c_double()
    eng._check(eng.lib.sabr_bench_mufu_peak(eng.handle, C.byref(v)))
    return v.value


def pipe_roofline(units_per_s, instr_per_unit, peak_tinstr_per_s, pipe, source):
    """A kernel's pipe occupancy: units/s x (ncu-counted) lane instructions of
    that pipe per unit, against the pipe's measured lane-instruction peak."""
    if not instr_per_unit or not peak_tinstr_per_s:
        return None
    a = units_per_s * instr_per_unit / 1e12
    return {"bound": pipe, "instr_per_unit": instr_per_unit, "achieved": a, "peak": peak_tinstr_per_s,
            "unit": "T lane-instr/s", "frac": a / peak_tinstr_per_s, "source": source}


def fp64_peak(eng):
    import ctypes as C

    v = C.c_double()
    eng._check(eng.lib.sabr_bench_fp64_peak(eng.handle, C.byref(v)))
    return v.value


def fp64_flops_per_eval():
    """FP64 FLOPs per cost-eval of the static level kernel (DFMA = 2), measured
    by ncu (profiles/fp64_per_eval.json); else the SURVEY 8(d) estimate."""
    p = os.path.join(ROOT, "profiles", "fp64_per_eval.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"flops": d["c2_flops_per_eval"], "source": d["source"], "instr": d.get("c2_fp64_instr_per_eval"),
                "dram_bytes_per_launch": d.get("c2_dram_bytes_per_launch"),
                "pipe_instr": d.get("c2_fp64_pipe_instr_per_eval"),
                "warp_instr": d.get("c2_warp_instr_per_eval")}
    # ~1180 FP64-pipe instructions per eval at m = 19 (upper bound,
    # counts one FLOP per instruction)
    return {"flops": 1180.0, "source": "SURVEY.md 8(d) estimate (FP64-pipe instr, m=19)"}


def secondary(eng, torch, dev, stream, peaks):
    """C4 (MC objective) and C3 (Case I) line items, measured once after a warm-up,
    each with the roofline of its dominant kernel (FP64 pipe, or the XU/MUFU
    pipe for the FP32 MC path) from profiles/fp64_per_eval.json's ncu counts."""
    import paper_2407_20713_b200 as pkg

    per = {}
    pth = os.path.join(ROOT, "profiles", "fp64_per_eval.json")
    if os.path.exists(pth):
        with open(pth) as f:
            per = json.load(f)
    fp64_lane_peak = peaks["fp64_tflops"] / 2  # DFMA = 2 FLOP: lane instructions / s
    src = "ncu lane instructions per unit (profiles/fp64_per_eval.json) x kernel units/s / measured pipe peak"
    out = {"peaks": {"fp64_tflops": peaks["fp64_tflops"], "mufu_tops": peaks["mufu_tops"],
                     "source": "sabr_bench_fp64_peak / sabr_bench_mufu_peak microbenchmarks (peak.cu), this run"}}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for precision, rng in (("fp64", "xoshiro"), ("fp32", "xoshiro"), ("fp64", "philox")):
        surf, fixed, sch, plan = c4_setup(levels=2)
        plan.precision = precision
        plan.rng = rng
        small = pkg.AnnealingSchedule(t0=2.0, cooling=0.5, chain_length=2, workers=32, t_min=1.5, seed=1)
        eng.calibrate_case2_T2(surf, None, small, plan, fixed)  # warm-up (jump tables, buffers)
        flush_l2(torch, dev)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        rep = eng.calibrate_case2_T2(surf, None, sch, plan, fixed)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        t = eng.last_timing()
        secs = e0.elapsed_time(e1) / 1e3
        steps_per_eval = 250
        ps = (rep.evals - 1) * plan.num_paths * steps_per_eval
        key = "c4_mc_calibration" + ("" if precision == "fp64" else "_fp32") + ("" if rng == "xoshiro" else "_philox")
        out[key] = {
            "metric": f"MC SABR path-steps/s (calibrate_case2_T2 objective, C4, {precision}, {rng} streams)",
            "unit": "path-steps/s", "value": ps / secs,
            "kernel_path_steps_per_s": t.path_steps / (t.kernel_ms / 1e3),
            "cost_evals": rep.evals - 1, "levels": 2, "chains": 32, "paths": plan.num_paths,
            "steps_per_path": steps_per_eval, "rng": plan.rng, "precision": precision, "seconds": secs,
            "final_cost": rep.final_cost, "mc_kernel_ms": t.kernel_ms, "mc_launches": t.kernel_launches}
        kps = t.path_steps / (t.kernel_ms / 1e3)
        if precision == "fp64":
            out[key]["roofline"] = pipe_roofline(kps, per.get("c4_fp64_pipe_instr_per_candidate_path_step"),
                                                 fp64_lane_peak, "fp64", src)
        else:
            out[key]["roofline"] = pipe_roofline(kps, per.get("c4_fp32_xu_instr_per_candidate_path_step"),
                                                 peaks["mufu_tops"], "xu (MUFU)", src)
    # C5: full Case II MC calibration on the 20x30 synthetic surface, one SA step of 2048 chains
    surf, bounds, sch, plan = c5_setup()
    for precision in ("fp64", "fp32"):
        plan.precision = precision
        eng.calibrate_case2_T2(surf, bounds, sch, plan, None)  # warm-up: jump tables, buffers
        flush_l2(torch, dev)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        rep = eng.calibrate_case2_T2(surf, bounds, sch, plan, None)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        t = eng.last_timing()
        secs = e0.elapsed_time(e1) / 1e3
        steps = t.path_steps / max(1, plan.num_paths * (rep.evals - 1))  # sum of per-slice steps
        out["c5_mc_calibration" + ("" if precision == "fp64" else "_fp32")] = {
            "metric": f"MC SABR path-steps/s (calibrate_case2_T2, full Case II, C5 20x30 surface, {precision})",
            "unit": "path-steps/s", "value": t.path_steps / secs,
            "kernel_path_steps_per_s": t.path_steps / (t.kernel_ms / 1e3),
            "cost_evals": rep.evals - 1, "levels": 1, "chains": sch.workers * sch.groups,
            "paths": plan.num_paths, "steps_per_path_all_slices": steps, "rng": plan.rng,
            "precision": precision, "seconds": secs, "final_cost": rep.final_cost,
            "sample": "one SA step (L=1, one level) of 2048 chains; C5 names 1e6 chains over 8 GPUs "
                      "(125000 per GPU, ~61x this sample per GPU-step)"}
        kps = t.path_steps / (t.kernel_ms / 1e3)
        k5 = "c5_mc_calibration" + ("" if precision == "fp64" else "_fp32")
        if precision == "fp64":
            out[k5]["roofline"] = pipe_roofline(kps, per.get("c5_fp64_pipe_instr_per_candidate_path_step"),
                                                fp64_lane_peak, "fp64", src)
        else:
            out[k5]["roofline"] = pipe_roofline(kps, per.get("c5_fp32_xu_instr_per_candidate_path_step"),
                                                peaks["mufu_tops"], "xu (MUFU)", src)
    # MC European pricing in the paper's shape (SSabr, 2^24 paths, 123 + 1 steps of
    # 1/250 to T = 0.4959), through price_european_batch; the paper's GTX470 did 2.18e8 (FP64) and
    # 1.62e9 (FP32) path-steps/s on this workload
    p_reg = pkg.StaticSabrParams(0.375162, 0.999999, 0.331441, -0.999999)
    for precision in ("fp64", "fp32"):
        plan = pkg.SimulationPlan(num_paths=1 << 24, seed=5, rng="xoshiro", precision=precision)
        eng.price_european_batch(p_reg, 2257.37, [2257.37], 0.018196, 0.034516, 0.495890, plan)
        flush_l2(torch, dev)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        est = eng.price_european_batch(p_reg, 2257.37, [2257.37], 0.018196, 0.034516, 0.495890, plan)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        secs = e0.elapsed_time(e1) / 1e3
        ps = float(plan.num_paths) * 124
        out["mc_european_pricing" + ("" if precision == "fp64" else "_fp32")] = {
            "metric": f"MC SABR path-steps/s (price_european_batch, 2^24 paths x 124 steps, {precision})",
            "unit": "path-steps/s", "value": ps / secs, "seconds": secs, "price": est[0].value,
            "std_error": est[0].std_error, "paper_gtx470_path_steps_per_s": 2.18e8 if precision == "fp64" else 1.62e9}
        if precision == "fp64":
            out["mc_european_pricing"]["roofline"] = pipe_roofline(
                ps / secs, per.get("mc_single_fp64_pipe_instr_per_path_step"), fp64_lane_peak, "fp64",
                src + " (whole call: simulate + reduce)")
        else:
            out["mc_european_pricing_fp32"]["roofline"] = pipe_roofline(
                ps / secs, per.get("mc_single_fp32_xu_instr_per_path_step"), peaks["mufu_tops"], "xu (MUFU)",
                src + " (whole call: simulate + reduce)")
    # C1 (BASELINE.json configs[0]): the reference's own CPU-sized case, static T_I on one EURO STOXX 50
    # slice with the acceptance schedule (32 chains, 412 levels, 1,000,001 evals): latency-bound on a GPU
    eq = pkg.parse_surface(os.path.join(ROOT, "tests", "data", "eurostoxx50.csv"))
    s1 = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=32, t_min=1e-7, seed=1)
    eng.calibrate_static_T1(eq, 0, None, s1, None)
    runs = []
    for _ in range(5):  # a ~10 ms call: the median of five
        e0.record(stream)
        rep = eng.calibrate_static_T1(eq, 0, None, s1, None)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        runs.append(e0.elapsed_time(e1) / 1e3)
    secs = float(np.median(runs))
    out["c1_static_calibration"] = {"metric": "calibrate_static_T1 wall time, C1 (EURO STOXX 50 slice 0, 32 chains)",
                                    "unit": "s", "value": secs, "cost_evals": rep.evals - 1,
                                    "cost_evals_per_s": (rep.evals - 1) / secs, "final_cost": rep.final_cost,
                                    "runs_s": runs, "statistic": "median of 5"}
    # C3: Case I joint calibration, EUR/USD, beta = 1 (acceptance.cpp:317-339 schedule, 1e5 chains)
    fx = pkg.parse_surface(os.path.join(ROOT, "tests", "data", "eurusd.csv"))
    s3 = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=12_500, groups=8, t_min=1e-7,
                               seed=1, max_evals=10 ** 12)
    eng.calibrate_dynamic_case1_T1(fx, None, pkg.AnnealingSchedule(t0=2, cooling=0.5, workers=64, t_min=1,
                                                                   seed=1), {"beta": 1.0})
    e0.record(stream)
    rep = eng.calibrate_dynamic_case1_T1(fx, None, s3, {"beta": 1.0})
    e1.record(stream)
    torch.cuda.synchronize(dev)
    secs = e0.elapsed_time(e1) / 1e3
    out["c3_case1_calibration"] = {"metric": "SA cost-evals/s, Case I (Eq. 8) joint calibration, EUR/USD, 1e5 chains",
                                   "unit": "cost-evals/s", "value": (rep.evals - 1) / secs, "seconds": secs,
                                   "mean_rel_error": rep.mean_rel_error}
    if per.get("c3_flops_per_eval"):
        a = (rep.evals - 1) / secs * per["c3_flops_per_eval"] / 1e12
        out["c3_case1_calibration"]["roofline"] = {
            "bound": "fp64", "achieved": a, "peak": peaks["fp64_tflops"], "unit": "TFLOP/s",
            "frac": a / peaks["fp64_tflops"], "flops_per_eval": per["c3_flops_per_eval"],
            "source": "ncu DFMA x2 + DADD + DMUL per eval (profiles/fp64_per_eval.json), whole calibration"}
        if per.get("c3_fp64_pipe_instr_per_eval"):
            out["c3_case1_calibration"]["roofline"]["fp64_pipe"] = pipe_roofline(
                (rep.evals - 1) / secs, per["c3_fp64_pipe_instr_per_eval"], fp64_lane_peak, "fp64", src)
    return out


def host_info():
    """CPU model, logical CPUs and glibc of the host running the CPU arms."""
    import platform

    model = platform.processor() or "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "glibc": "-".join(platform.libc_ver())}


def full_configs(eng, torch, dev, stream, peaks):
    """BASELINE configs C4 and C5 at their named sizes (bench.py --full-configs):
    * C4: calibrate_case2_T2 on the T=1 equity slice with static dynamics, 32
      chains x 100 steps per level, t_min 1e-7 (all 412 levels), 1e5 paths x
      250 steps per cost-eval;
    * C5: one SA step of 125,000 chains (1e6 chains over 8 GPUs, this GPU's
      share) of the full Case II calibration on the 20x30 surface in the
      default Case II box (calibration.cpp:46-60), 4096 paths per candidate."""
    import paper_2407_20713_b200 as pkg

    out = {}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn):
        flush_l2(torch, dev)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        r = fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        return r, e0.elapsed_time(e1) / 1e3

    surf, fixed, _, plan = c4_setup()
    sch = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=32, t_min=1e-7, seed=1,
                                max_evals=10 ** 12)
    rep, secs = timed(lambda: eng.calibrate_case2_T2(surf, None, sch, plan, fixed))
    t = eng.last_timing()
    out["c4_full_calibration"] = {
        "metric": "calibrate_case2_T2 wall time and path-steps/s, C4 (whole calibration: 412 levels, 32 chains, "
                  "1e5 paths x 250 steps per cost-eval, fp64)",
        "unit": "path-steps/s", "value": t.path_steps / secs, "seconds": secs, "cost_evals": rep.evals - 1,
        "path_steps": t.path_steps, "final_cost": rep.final_cost, "params": rep.params,
        "kernel_path_steps_per_s": t.path_steps / (t.kernel_ms / 1e3)}
    for precision in ("fp64", "fp32"):
        surf5, _, sch5, plan5 = c5_setup(chains=125_000)
        plan5.precision = precision
        rep, secs = timed(lambda: eng.calibrate_case2_T2(surf5, None, sch5, plan5, None))
        t = eng.last_timing()
        out["c5_per_gpu_step" + ("" if precision == "fp64" else "_fp32")] = {
            "metric": f"MC SABR path-steps/s, C5 per-GPU SA step (125,000 chains, default Case II box, {precision})",
            "unit": "path-steps/s", "value": t.path_steps / secs, "seconds": secs, "cost_evals": rep.evals - 1,
            "path_steps": t.path_steps, "kernel_path_steps_per_s": t.path_steps / (t.kernel_ms / 1e3),
            "note": "proposals outside the Case II feasibility grid are skipped without an eval "
                    "(annealer.cpp:122), as in the reference"}
    return out


def cpu_baseline(fx):
    """The compiled reference (oracle/_ref) on the host cores: the headline
    C2 sample at all threads (the line's cpu_baseline), plus the BASELINE.md
    section 3 matrix - C1 (whole run), C2, C3, C4 and C5 at 1 thread and at all
    threads, each a bounded sample (about 20 s in total)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracles import Ref, have_ref

    import paper_2407_20713_b200 as pkg

    if not have_ref():
        return {"value": None, "unit": "cost-evals/s", "cores": 0, "kind": "reference",
                "sample": "oracle/_ref not built"}
    ref = Ref()
    threads = ref.max_threads()

    def timed(fn):
        t0 = time.perf_counter()
        out = fn()
        return out, time.perf_counter() - t0

    sch = c2_schedule(1, max_evals=2 * 10 ** 7 + 1)
    sch.omp_threads = threads
    rep, secs = timed(lambda: ref.calibrate_static_T1(fx, 0, None, sch, None))
    line = {"value": (rep.evals - 1) / secs, "unit": "cost-evals/s", "cores": threads, "kind": "reference",
            "sample": f"calibrate_static_T1(eurusd slice 0), C2 schedule capped at max_evals=2e7 "
                      f"(first 2 levels, {rep.evals - 1} evals, {secs:.1f} s)"}
    eq = pkg.parse_surface(os.path.join(ROOT, "tests", "data", "eurostoxx50.csv"))
    matrix = {}
    for n in sorted({1, threads}):
        row = {}
        # C1: the reference's own CPU-sized case, the whole acceptance-schedule run
        s1 = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=32, t_min=1e-7, seed=1)
        s1.omp_threads = n
        r, t = timed(lambda: ref.calibrate_static_T1(eq, 0, None, s1, None))
        row["c1_static_calibration_s"] = t
        row["c1_cost_evals_per_s"] = (r.evals - 1) / t
        # C2: the C2 schedule on one EUR/USD slice, first level (1e7 evals; 1e6 at 1 thread)
        s2 = c2_schedule(1, max_evals=(10 ** 7 if n > 1 else 10 ** 6) + 1)
        s2.omp_threads = n
        r, t = timed(lambda: ref.calibrate_static_T1(fx, 0, None, s2, None))
        row["c2_cost_evals_per_s"] = (r.evals - 1) / t
        # C3: Case I joint calibration, acceptance schedule, beta = 1 (1e6 evals)
        s3 = pkg.AnnealingSchedule(t0=2.0, cooling=0.96, chain_length=100, workers=32, t_min=1e-7, seed=1)
        s3.omp_threads = n
        r, t = timed(lambda: ref.calibrate_dynamic_case1_T1(fx, None, s3, {"beta": 1.0}))
        row["c3_cost_evals_per_s"] = (r.evals - 1) / t
        # C4: one MC cost-eval (case2_mc_cost, 1e5 paths x 250 steps, static dynamics)
        surf4, _, _, plan4 = c4_setup()
        plan4.workers = n
        P4 = np.array([[0.30, 1.0, -0.45, 0.0, 0.0, 0.9, 0.0, 0.0, 0.0, 0.0, 1.0]])
        _, t = timed(lambda: ref.cost_case2_mc(surf4, P4, plan4))
        row["c4_path_steps_per_s"] = 1e5 * 250 / t
        # C5: one MC cost-eval on the 20x30 surface (4096 paths, 13130 steps per path)
        surf5 = pkg.parse_surface(os.path.join(ROOT, "tests", "data", "synth20x30.csv"))
        plan5 = pkg.SimulationPlan(num_paths=4096, dt=1 / 250, seed=1, rng="xoshiro")
        plan5.workers = n
        P5 = np.array([FX_CASE2 + [5.0]])
        _, t = timed(lambda: ref.cost_case2_mc(surf5, P5, plan5))
        row["c5_path_steps_per_s"] = 4096 * 13130 / t
        matrix[f"threads_{n}"] = row
    line["matrix"] = matrix
    line["host"] = host_info()
    return line


def run_reference(args):
    """--impl reference: the compiled reference CPU implementation, all host threads."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracles import Ref, have_ref

    import paper_2407_20713_b200.api as api

    if not have_ref():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libsabr_ref.so not built"}))
        return
    ref = Ref()
    threads = ref.max_threads()
    from oracles import ref_parse_surface

    fx = ref_parse_surface(os.path.join(ROOT, "tests", "data", "eurusd.csv"))
    sch = c2_schedule(world, max_evals=10 ** 7 + 1)
    sch.omp_threads = threads

    def step(sl):
        t0 = time.perf_counter()
        rep = ref.calibrate_static_T1(fx, sl, None, sch, None)
        return rep.evals - 1, time.perf_counter() - t0

    for i in range(args.warmup):
        step(i % 4)
    ev, secs = 0, 0.0
    for i in range(args.steps):
        e, s = step(i % 4)
        ev += e
        secs += s
    value = ev / secs
    print(json.dumps({
        "impl": "reference",
        "metric": "SA cost-evals/s, static Hagan/Obloj (Eq. 7) calibration, EUR/USD surface, 1e5 chains/GPU",
        "value": value, "unit": "cost-evals/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "reference fixture proj/data/eurusd.csv",
        "config": {"workload": "C2 (bounded CPU sample: each step = calibrate_static_T1 on one EUR/USD slice "
                               f"with the C2 schedule capped at max_evals=1e7, {threads} OpenMP threads)"},
        "cpu_baseline": {"value": value, "unit": "cost-evals/s", "cores": threads, "kind": "reference",
                         "sample": "1e7 cost-evals per step (first level of the C2 schedule)"},
        "e2e": {"value": value, "unit": "cost-evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def launch_plan(gpus, env, argv):
    """How `bench.py --gpus N` runs: ("run", None) in this process, ("exec",
    cmd) to re-launch itself under torch.distributed.run with N ranks (when
    started without a launcher), or ("error", msg) when a launcher's
    WORLD_SIZE disagrees with --gpus (--gpus is authoritative)."""
    if gpus < 1:
        return "error", f"--gpus must be >= 1 (got {gpus})"
    world = env.get("WORLD_SIZE")
    if world is None:
        if gpus == 1:
            return "run", None
        port = env.get("MASTER_PORT", "29531")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(argv)
        return "exec", cmd
    if int(world) != gpus:
        return "error", f"WORLD_SIZE={world} but --gpus {gpus}: launch one rank per GPU"
    return "run", None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--full-configs", action="store_true",
                    help="also run C4 as a whole calibration and C5 at its per-GPU size (about 3 minutes)")
    args = ap.parse_args()
    what, detail = launch_plan(args.gpus, os.environ, sys.argv[1:])
    if what == "error":
        print(f"bench.py: {detail}", file=sys.stderr)
        sys.exit(2)
    if what == "exec":
        os.execv(detail[0], detail)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
