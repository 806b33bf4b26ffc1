"""Summarise one kernel of an `ncu --set full` report into profiles/ JSON.

usage: python tools/ncu_summary.py REPORT.ncu-rep OUT.json [limbs] [traffic.json] [bytes_per_unit]
Reads the raw page (ncu -i ... --page raw --csv) of the first captured kernel,
keeps the metrics DESIGN.md argues from, the PC-sampling stall histogram and,
given the limb count of the launch, the DRAM bytes per limb (written also to
traffic.json, which bench.py reports as roofline.traffic)."""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
    return float(v) * scale


def main():
    rep, out = sys.argv[1], sys.argv[2]
    limbs = int(sys.argv[3]) if len(sys.argv) > 3 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    gi = hdr.index("launch__grid_size")
    # several launches may be captured: summarise the largest (the benchmarked one)
    val = max(rows[2:], key=lambda r: int(float(r[gi].replace(",", "") or 0)))
    col = {k: i for i, k in enumerate(hdr)}
    res = {}
    for k in KEYS:
        if k in col:
            res[k] = (val[col[k]] + " " + units[col[k]]).strip()
    pre = "smsp__pcsamp_warps_issue_stalled_"
    stalls = {k[len(pre):]: int(float(val[i].replace(",", "") or 0)) for k, i in col.items()
              if k.startswith(pre) and not k.endswith("_not_issued")}
    res["pc_sampling_stalls"] = dict(sorted(((k, v) for k, v in stalls.items() if v), key=lambda kv: -kv[1])[:10])
    if limbs:
        rd = to_bytes(val[col["dram__bytes_read.sum"]], units[col["dram__bytes_read.sum"]])
        wr = to_bytes(val[col["dram__bytes_write.sum"]], units[col["dram__bytes_write.sum"]])
        res["limbs"] = limbs
        res["dram_bytes_per_limb"] = (rd + wr) / limbs
        res["algorithmic_bytes_per_limb"] = int(sys.argv[5]) if len(sys.argv) > 5 else 2 * 8 * 8192
    json.dump(res, open(out, "w"), indent=1)
    if limbs and len(sys.argv) > 4:
        name = res["Kernel Name"].replace("void ", "").replace("unnamed>::", "").split("(")[0]
        def pct(k):
            try:
                return round(float(val[col[k]].replace(",", "")) / 100.0, 4)
            except (KeyError, ValueError):
                return None
        n_dim = 32768 if "c4" in name else 8192
        rec = {"kernel": name, "N": n_dim, "source": f"{out} (ncu --set full, {limbs}-unit launch)",
               "bytes_per_limb": res["dram_bytes_per_limb"],
               "fmaheavy_frac": pct("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
               "alu_frac": pct("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
               "issue_frac": pct("smsp__issue_active.avg.pct_of_peak_sustained_active")}
        if "ks_inner" in name:
            rec["bytes_per_rotation"] = rec.pop("bytes_per_limb")
        json.dump(rec, open(sys.argv[4], "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
