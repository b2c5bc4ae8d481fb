"""Key counters of `ncu --set full` captures: issue, warps, pipe use, stall
reasons per issued instruction and the opcode mix (profiles/<round>_ncu_stalls.txt).

    python tools/ncu_stalls.py gpurun_out/full_sa.ncu-rep [...] > profiles/r02d_ncu_stalls.txt"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_active.avg.per_cycle_active", "smsp__warps_eligible.avg.per_cycle_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2]


def main(reps):
    for rep in reps:
        h, units, v = raw(rep)
        d = dict(zip(h, v))
        print(f"== {rep}: {d.get('Kernel Name', '')[:110]}")
        for k in KEYS:
            if k in d:
                print(f"  {k:70s} {d[k]}")
        st = sorted(((float(d[k]), k) for k in h if k.startswith("smsp__average_warps_issue_stalled_")
                     and k.endswith("_per_issue_active.ratio") and d[k] not in ("", "n/a")), reverse=True)
        print("  stalls per issued instruction:")
        for val, k in st:
            if val >= 0.02:
                print(f"    {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:28s} {val:.3f}")


if __name__ == "__main__":
    main(sys.argv[1:])
