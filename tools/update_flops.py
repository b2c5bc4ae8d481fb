"""Refresh profiles/fp64_per_eval.json from a round's ncu metric CSVs
(gpurun_out/ncu_metrics_{sa,case1,t2,mc}.csv) and copy them to profiles/<tag>_*."""
import json
import os
import shutil
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summarise  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def per(path, prefix, units, pick=-1):
    mets = [m for k, m in summarise(path).items() if k.startswith(prefix)]
    m = mets[pick]
    g = {k: sum(v) / len(v) for k, v in m.items()}
    dfma = g["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]
    dadd = g["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
    dmul = g["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"]
    pipe = g.get("smsp__inst_executed_pipe_fp64.sum")  # warp instructions of the FP64 pipe
    warp_inst = g.get("smsp__inst_executed.sum")
    xu = g.get("smsp__inst_executed_pipe_xu.sum")  # warp instructions of the XU (MUFU) pipe
    return ((2 * dfma + dadd + dmul) / units, (dfma + dadd + dmul) / units,
            g["dram__bytes_read.sum"] + g["dram__bytes_write.sum"], g["gpu__time_duration.sum"],
            None if pipe is None else 32 * pipe / units, None if warp_inst is None else warp_inst / units,
            None if xu is None else 32 * xu / units)


def main(tag, copy=("sa", "case1", "t2", "t2_fp32", "mc", "mc_fp32", "c5", "c5_fp32")):
    src = os.path.join(ROOT, "gpurun_out")
    sa = per(os.path.join(src, "ncu_metrics_sa.csv"), ("sa_level_multi_kernel<0", "sa_level_kernel<0"), 1e7)
    c1 = per(os.path.join(src, "ncu_metrics_case1.csv"), ("sa_level_multi_kernel<1", "sa_level_kernel<1"), 1e7)
    t2 = per(os.path.join(src, "ncu_metrics_t2.csv"), "mc_tile_kernel<8", 32 * 1e5 * 250)
    mc = per(os.path.join(src, "ncu_metrics_mc.csv"), "mc_tile_kernel<1", (1 << 20) * 124)
    d = {"source": f"ncu smsp__sass_thread_inst_executed_op_{{dfma,dadd,dmul}}_pred_on.sum (DFMA = 2 FLOP) "
                   f"per unit, profiles/{tag}_ncu_metrics_*.csv (tools/profile_kernels.py)",
         "c2_flops_per_eval": sa[0], "c2_fp64_instr_per_eval": sa[1], "c2_dram_bytes_per_launch": sa[2],
         "c2_level_kernel_ns": sa[3], "c2_fp64_pipe_instr_per_eval": sa[4],
         "c2_warp_instr_per_eval": sa[5],
         "c3_flops_per_eval": c1[0], "c3_fp64_instr_per_eval": c1[1], "c3_dram_bytes_per_launch": c1[2],
         "c3_level_kernel_ns": c1[3],
         "c4_flops_per_candidate_path_step": t2[0], "c4_fp64_instr_per_candidate_path_step": t2[1],
         "c4_dram_bytes_per_launch": t2[2], "c4_mc_kernel_ns": t2[3],
         "c4_fp64_pipe_instr_per_candidate_path_step": t2[4],
         "mc_single_flops_per_path_step": mc[0], "mc_single_fp64_instr_per_path_step": mc[1],
         "mc_single_fp64_pipe_instr_per_path_step": mc[4]}
    f32 = os.path.join(src, "ncu_metrics_t2_fp32.csv")
    if os.path.exists(f32):  # the FP32 MC path: MUFU (XU) instructions per candidate-path-step
        # C4 FP32 runs 16 candidates per thread (time-invariant rows), earlier builds 8
        try:
            t2f = per(f32, "mc_tile_kernel_f32<16", 32 * 1e5 * 250)
        except IndexError:
            t2f = per(f32, "mc_tile_kernel_f32<8", 32 * 1e5 * 250)
        d["c4_fp32_xu_instr_per_candidate_path_step"] = t2f[6]
        d["c4_fp32_mc_kernel_ns"] = t2f[3]
        d["c4_fp32_warp_instr_per_candidate_path_step"] = t2f[5]
    c3 = os.path.join(src, "ncu_metrics_case1.csv")
    if os.path.exists(c3):
        d["c3_fp64_pipe_instr_per_eval"] = c1[4]
        d["c3_warp_instr_per_eval"] = c1[5]
    # C5 (one SA step of tools/profile_kernels.py c5: a single MC launch whose
    # candidate-path-steps the tool prints) and single-candidate FP32 pricing
    for name, csvf, prefix, log in (("c5", "ncu_metrics_c5.csv", "mc_tile_kernel<", "prof_c5.log"),
                                    ("c5_fp32", "ncu_metrics_c5_fp32.csv", "mc_tile_kernel_f32<", "prof_c5_fp32.log")):
        pc, pl = os.path.join(src, csvf), os.path.join(src, log)
        if not (os.path.exists(pc) and os.path.exists(pl)):
            continue
        units = None
        for line in open(pl):
            if line.startswith("path_steps"):
                units = float(line.split()[1])
        if units:
            r = per(pc, prefix, units)
            if name == "c5":
                d["c5_fp64_pipe_instr_per_candidate_path_step"] = r[4]
                d["c5_flops_per_candidate_path_step"] = r[0]
            else:
                d["c5_fp32_xu_instr_per_candidate_path_step"] = r[6]
    mf = os.path.join(src, "ncu_metrics_mc_fp32.csv")
    if os.path.exists(mf):
        r = per(mf, "mc_tile_kernel_f32<1", (1 << 20) * 124)
        d["mc_single_fp32_xu_instr_per_path_step"] = r[6]
    with open(os.path.join(ROOT, "profiles", "fp64_per_eval.json"), "w") as f:
        json.dump(d, f, indent=1)
    for m in copy:
        p = os.path.join(src, f"ncu_metrics_{m}.csv")
        if os.path.exists(p):
            shutil.copy(p, os.path.join(ROOT, "profiles", f"{tag}_ncu_metrics_{m}.csv"))
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:3] and [sys.argv[2].split(",")]))
