#!/bin/bash
# forward NTT launch of bench.py's roofline: stall samples per barrier phase
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ntt_fwd3 -s 4 -c 1 -o gpurun_out/fwd_full -f \
    python tools/ntt_once.py > /dev/null 2>&1
python - <<'PY' > gpurun_out/fwd_seg_stalls.txt
import csv, io, re, subprocess, collections
out = subprocess.run(["ncu", "-i", "gpurun_out/fwd_full.ncu-rep", "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
si = h.index("Source"); smp = h.index("Warp Stall Sampling (All Samples)"); ni = h.index("Warp Stall Sampling (Not-issued Samples)")
seg = 0; tot = collections.Counter(); nis = collections.Counter(); top = collections.defaultdict(list)
for r in rows[2:]:
    src = r[si].strip()
    if src.startswith("BAR"): seg += 1
    a = int(r[smp] or 0); b = int(r[ni] or 0)
    tot[seg] += a; nis[seg] += b
    top[seg].append((a, src))
T = sum(tot.values())
for k in sorted(tot):
    print(f"phase {k}: samples {tot[k]} ({100*tot[k]/T:.1f}%), not-issued {nis[k]}")
    for a, src in sorted(top[k], reverse=True)[:6]:
        print(f"    {a:6d}  {src}")
PY
rm -f gpurun_out/fwd_full.ncu-rep
cat gpurun_out/fwd_seg_stalls.txt
