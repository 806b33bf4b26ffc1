#!/bin/bash
# bench lines with the k_ks_plan roofline, the ncu --set full capture of that launch, and
# the cfg5 end-to-end timeline
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
timeout 600 python bench.py --config cfg5 --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "cfg5 rc $?"
HGM_TRACE=1 timeout 300 python tools/e2e_breakdown5.py 32 > gpurun_out/e2e5.txt 2>&1; echo "e2e5 rc $?"; tail -25 gpurun_out/e2e5.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ks_plan -s 1 -c 1 -o gpurun_out/plan_full -f \
    python tools/plan_once.py > gpurun_out/ncu_plan_full.log 2>&1; echo "ncu plan rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ntt_fwd3 -s 4 -c 1 -o gpurun_out/ntt_full -f \
    python tools/ntt_once.py > gpurun_out/ncu_ntt_full.log 2>&1; echo "ncu ntt rc $?"
