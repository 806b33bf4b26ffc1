"""Per-phase report of the heaviest launch in an ncu SASS source-page CSV that may
hold several launches: python tools/phase_report.py gpurun_out/ntt_ph_fwd.csv"""
import csv
import subprocess
import sys
import tempfile

rows = list(csv.reader(open(sys.argv[1])))
blocks, cur, hdr = [], None, None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = []
        blocks.append((r, cur))
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if cur is not None and len(r) > 5:
        cur.append(r)
ie = hdr.index("Instructions Executed")
kr, b = max(blocks, key=lambda bl: sum(int(x[ie] or 0) for x in bl[1]))
with tempfile.NamedTemporaryFile("w", suffix=".csv", delete=False) as f:
    w = csv.writer(f)
    w.writerow(kr)
    w.writerow(hdr)
    for r in b:
        w.writerow(r)
print(kr[1][:80])
subprocess.run([sys.executable, "tools/sass_phases.py", f.name], check=True)
