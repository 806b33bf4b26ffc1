"""Metrics and the executed SASS opcode mix of one ncu --set full report.

usage: python tools/kernel_mix.py REPORT.ncu-rep [units]
Prints duration, DRAM bytes, pipe utilisation, issue activity, warps, stall
top-5, and executed warp instructions by opcode (per `units` if given, e.g. the
number of coefficients or butterflies the launch processed)."""
import collections
import csv
import io
import re
import subprocess
import sys


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    return {k: (v[i], u[i]) for i, k in enumerate(h)}


def mix(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    si, ei = h.index("Source"), h.index("Instructions Executed")
    c = collections.Counter()
    for r in rows[2:]:
        op = re.sub(r"^@!?U?P\w+\s+", "", r[si].strip()).split()
        if op:
            c[op[0]] += int(r[ei] or 0)
    return c


def main():
    rep = sys.argv[1]
    units = float(sys.argv[2]) if len(sys.argv) > 2 else None
    m = raw(rep)
    keys = ["Kernel Name", "launch__grid_size", "launch__registers_per_thread", "gpu__time_duration.sum",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum"]
    for k in keys:
        if k in m:
            print(f"{k:64s} {m[k][0]} {m[k][1]}")
    pre = "smsp__pcsamp_warps_issue_stalled_"
    st = {k[len(pre):]: float(v[0].replace(",", "") or 0) for k, v in m.items()
          if k.startswith(pre) and not k.endswith("_not_issued")}
    print("stalls:", dict(sorted(st.items(), key=lambda kv: -kv[1])[:6]))
    c = mix(rep)
    tot = sum(c.values())
    d = units or 1.0
    print(f"warp instructions {tot}" + (f" = {tot / d:.2f} per unit" if units else ""))
    for op, n in c.most_common(18):
        print(f"  {op:20s} {n / d:10.3f}")


if __name__ == "__main__":
    main()
