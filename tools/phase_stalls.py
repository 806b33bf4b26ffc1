"""Stall samples and executed instructions of a kernel split at its barriers:
python tools/phase_stalls.py REPORT.ncu-rep  (ncu --set full --import-source on)."""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
si, ns, ei = h.index("Source"), h.index("# Samples"), h.index("Instructions Executed")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_")]
seg, S = 0, collections.defaultdict(collections.Counter)
for r in rows[2:]:
    if r[si].strip().startswith("BAR"):
        seg += 1
    S[seg]["samples"] += int(r[ns] or 0)
    S[seg]["inst"] += int(r[ei] or 0)
    S[seg]["static"] += 1
    for i in stall_cols:
        S[seg][h[i]] += int(float(r[i] or 0))
tot = sum(s["samples"] for s in S.values())
ti = sum(s["inst"] for s in S.values())
for k in sorted(S):
    s = S[k]
    top = sorted(((v, n) for n, v in s.items() if n.startswith("stall_")), reverse=True)[:6]
    print(f"phase {k}: {s['static']:5d} SASS lines, {100 * s['inst'] / ti:5.1f}% of executed instructions, "
          f"{100 * s['samples'] / tot:5.1f}% of samples;",
          ", ".join(f"{n[6:]} {round(100 * v / max(1, s['samples']))}%" for v, n in top))
