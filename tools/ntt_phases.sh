#!/bin/bash
# ncu --set full of the 1184-limb forward and inverse NTT launches (tools/ntt_once.py),
# then the per-phase stall/instruction split of each (tools/sass_phases.py).  Run under gpurun.
set -e
python tools/ntt_once.py > gpurun_out/ntt_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_ntt_(fwd|inv)3" -c 10 -o gpurun_out/ntt_ph python tools/ntt_once.py > gpurun_out/ncu_ntt_ph.log 2>&1
for k in fwd inv; do
  ncu -i gpurun_out/ntt_ph.ncu-rep --page source --csv --print-source sass -k regex:k_ntt_${k}3 > gpurun_out/ntt_ph_${k}.csv 2>/dev/null || true
done
echo done
