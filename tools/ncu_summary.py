"""Summarise an `ncu --metrics ... --csv` launch list per kernel (mean over launches)."""
import collections
import csv
import sys


def summarise(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            k = d["Kernel Name"].split("(")[0].replace("void ", "").split("::")[-1]
            out.setdefault(k, collections.defaultdict(list))[d["Metric Name"]].append(
                float(d["Metric Value"].replace(",", "")))
    return out


if __name__ == "__main__":
    for path in sys.argv[1:]:
        print("==", path)
        for k, mets in summarise(path).items():
            n = len(next(iter(mets.values())))
            g = {m: sum(v) / len(v) for m, v in mets.items()}
            print(f"  {k} x{n}: time {g.get('gpu__time_duration.sum', 0)/1e3:.1f} us, "
                  f"fp64 pipe {g.get('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active', 0):.1f}%, "
                  f"warps {g.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):.1f}%, "
                  f"regs {g.get('launch__registers_per_thread', 0):.0f}, "
                  f"dfma {g.get('smsp__sass_thread_inst_executed_op_dfma_pred_on.sum', 0):.4g} "
                  f"dadd {g.get('smsp__sass_thread_inst_executed_op_dadd_pred_on.sum', 0):.4g} "
                  f"dmul {g.get('smsp__sass_thread_inst_executed_op_dmul_pred_on.sum', 0):.4g} "
                  f"inst {g.get('smsp__inst_executed.sum', 0):.4g} "
                  f"dram {g.get('dram__bytes_read.sum', 0) + g.get('dram__bytes_write.sum', 0):.4g}")
