#!/bin/bash
# launch list of the bench step and an ncu --set full capture of one k_ks_plan launch
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/plan_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_plan_bench.log 2>&1; echo "ncu launches rc $?"
python tools/launch_shares.py gpurun_out/plan_launches.csv > gpurun_out/plan_launches_shares.txt; head -14 gpurun_out/plan_launches_shares.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ks_plan -s 1 -c 1 -o gpurun_out/plan_full -f \
    python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --instances 1024 > gpurun_out/ncu_plan_full.log 2>&1; echo "ncu plan rc $?"
python tools/ncu_summary.py gpurun_out/plan_full.ncu-rep gpurun_out/plan_full.json; cat gpurun_out/plan_full.json
