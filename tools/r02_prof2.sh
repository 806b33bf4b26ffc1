#!/bin/bash
# ncu --set full of the inverse NTT launch bench.py times, and of one in-step launch of the fused
# ModDown kernels and the Q->B conversion (256-instance cloud step)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ntt_inv3 -s 2 -c 1 -o gpurun_out/inv_full -f \
    python tools/ntt_once.py > gpurun_out/ncu_inv_full.log 2>&1; echo "ncu inv rc $?"
K=256 KERNELS="k_ntt_fwd_io k_ntt_inv_io k_q_to_b2" timeout 1500 bash tools/prof_kernels_full.sh
