#!/bin/bash
# tools/prof_kernels_full.sh, then the metric / opcode summaries (tools/kernel_mix.py)
# written to gpurun_out/mix_<kernel>.txt; the bulky reports are deleted (the
# gpurun_out merge is capped at 64 MiB) unless KEEP names one to keep.
bash tools/prof_kernels_full.sh
for r in gpurun_out/full_*.ncu-rep; do
  k=$(basename $r .ncu-rep); k=${k#full_}
  python tools/kernel_mix.py $r > gpurun_out/mix_$k.txt 2>&1
  [ "$k" = "$KEEP" ] || rm -f $r
done
ls gpurun_out/
