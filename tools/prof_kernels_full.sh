#!/bin/bash
# ncu --set full of one launch of each named kernel inside a 1024-instance cloud
# step (after a warm-up step), for the source-level instruction mix.
K=${K:-1024}
python tools/profile_step.py $K > gpurun_out/prof_plain.txt 2>&1
SKIP=$(sed -n 's/.*skip=\([0-9]*\).*/\1/p' gpurun_out/prof_plain.txt)
for k in ${KERNELS:-k_lincomb k_q_to_b k_tensor_acc k_ks_inner k_ntt_inv3 k_ntt_fwd_io k_ntt_inv_io}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip-before-match $SKIP -s 1 -c 1 \
     -o gpurun_out/full_$k -f python tools/profile_step.py $K > gpurun_out/ncu_full_$k.log 2>&1
  echo "$k rc $?"
done
