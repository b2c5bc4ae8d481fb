"""Opcode mix + top stall sites of an ncu --set full report (--page source --print-source sass)."""
import collections
import csv
import io
import re
import subprocess
import sys


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]


def main(rep, units, top=25):
    data = load(rep)
    tot = sum(int(d["Instructions Executed"] or 0) for d in data)
    samp = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
    op, opsamp = collections.Counter(), collections.Counter()
    for d in data:
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", d["Source"])
        name = m.group(2) if m else "?"
        op[name] += int(d["Instructions Executed"] or 0)
        opsamp[name] += int(d["Warp Stall Sampling (All Samples)"] or 0)
    print(f"warp instructions {tot:.4g} ({tot / units:.1f} per unit-warp), stall samples {samp}")
    for k, v in op.most_common(top):
        print(f"  {k:10s} {v / tot * 100:6.2f}% instr {opsamp[k] / samp * 100:6.2f}% samples  {v / units:7.2f}/unit")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]))
