"""Executed instructions of an NTT kernel split at its barriers (load / rounds /
store phases), per butterfly of the launch: python tools/ntt_segments.py REPORT limbs [logN]."""
import collections
import csv
import io
import re
import subprocess
import sys

rep, limbs = sys.argv[1], int(sys.argv[2])
logn = int(sys.argv[3]) if len(sys.argv) > 3 else 13
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
si, ei = h.index("Source"), h.index("Instructions Executed")
wb = (1 << (logn - 1)) * logn // 32 * limbs  # warp-butterflies of the launch
seg, segs = 0, collections.defaultdict(collections.Counter)
for r in rows[2:]:
    src = r[si].strip()
    if src.startswith("BAR"):
        seg += 1
    op = re.sub(r"^@!?U?P\w+\s+", "", src).split()
    if op:
        segs[seg][op[0]] += int(r[ei] or 0)
tot = sum(sum(c.values()) for c in segs.values())
print(f"{tot / wb:.2f} warp instructions per warp-butterfly")
for k in sorted(segs):
    c = segs[k]
    print(k, f"{sum(c.values()) / wb:.2f}", {o: round(v / wb, 2) for o, v in c.most_common(8)})
