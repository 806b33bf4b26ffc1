"""Per-kernel table from tools/prof_metrics.sh's ncu CSV (gpurun_out/metrics.csv)."""
import collections
import csv
import sys

KEYS = ["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, idi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    for r in data:
        per[(r[idi], r[ki])][r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    for (_, k), m in per.items():
        name = k.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "").replace("unnamed>::", "")
        a = agg[name]
        t = m["gpu__time_duration.sum"]
        a["n"] += 1
        a["t"] += t
        a["bytes"] += m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        for key in KEYS:
            a[key] += m[key] * t
        a["regs"] = m["launch__registers_per_thread"]
    tot = sum(a["t"] for a in agg.values())
    print(f"total {tot / 1e6:.2f} ms over {sum(int(a['n']) for a in agg.values())} launches")
    print(f"{'kernel':30s} {'n':>4s} {'share':>6s} {'avg_us':>8s} {'GB/s':>7s} {'dram%':>6s} {'fmaH%':>6s} {'alu%':>6s} "
          f"{'issue%':>6s} {'warps%':>6s} regs")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["t"]):
        t = a["t"]
        print(f"{k[:30]:30s} {int(a['n']):4d} {100 * t / tot:6.1f} {t / a['n'] / 1e3:8.1f} {a['bytes'] / t:7.0f} "
              + " ".join(f"{a[key] / t:6.1f}" for key in KEYS) + f" {int(a['regs'])}")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/metrics.csv")
