#!/bin/bash
# ncu --set full of the benchmarked inverse NTT launch (4736 limbs), segment split on the box
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ntt_inv3 -s 1 -c 1 -o gpurun_out/inv_full -f \
    python tools/ntt_once.py > gpurun_out/ncu_inv_full.log 2>&1
python tools/kernel_mix.py gpurun_out/inv_full.ncu-rep > gpurun_out/mix_inv3.txt 2>&1
python tools/ntt_segments.py gpurun_out/inv_full.ncu-rep 4736 > gpurun_out/seg_inv3.txt 2>&1
rm -f gpurun_out/inv_full.ncu-rep
cat gpurun_out/seg_inv3.txt; grep -E "grid|duration|fmaheavy|alu|issue|stalls" gpurun_out/mix_inv3.txt
