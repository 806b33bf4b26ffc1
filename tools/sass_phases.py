"""Split an ncu SASS source page (ncu -i R --page source --csv --print-source sass)
into barrier-delimited phases: warp-stall samples and executed instructions per phase."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
si, ii, ni = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
phases, cur = [], {"samples": 0, "inst": 0, "n": 0, "first": None, "ops": {}}
for r in rows[2:]:
    if len(r) <= max(si, ii, ni):
        continue
    src = r[si].strip()
    op = src.split()[0] if src else ""
    if op.startswith("@"):
        op = src.split()[1]
    cur["samples"] += int(r[ii] or 0)
    cur["inst"] += int(r[ni] or 0)
    cur["n"] += 1
    cur["first"] = cur["first"] or src
    base = op.split(".")[0]
    cur["ops"][base] = cur["ops"].get(base, 0) + int(r[ni] or 0)
    if base == "BAR":
        phases.append(cur)
        cur = {"samples": 0, "inst": 0, "n": 0, "first": None, "ops": {}}
phases.append(cur)
ts = sum(p["samples"] for p in phases) or 1
ti = sum(p["inst"] for p in phases) or 1
for k, p in enumerate(phases):
    top = sorted(p["ops"].items(), key=lambda kv: -kv[1])[:6]
    print(f"phase {k}: {p['n']:5d} sass  samples {100 * p['samples'] / ts:5.1f}%  inst {100 * p['inst'] / ti:5.1f}%  "
          + " ".join(f"{o}:{100 * v / ti:.1f}" for o, v in top))
