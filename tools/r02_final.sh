#!/bin/bash
# Final round-2 evidence (run under gpurun, one GPU; every step under its own timeout):
# GPU tests, smoke, both bench lines, the reference arm, the ncu launch list of the bench
# command and ncu --set full captures of the forward NTT, k_ks_inner and k_ks_plan
# launches bench.py's roofline times.
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest.log
tail -3 gpurun_out/gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
timeout 600 python bench.py --config cfg5 --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "cfg5 rc $?"
timeout 600 python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err; echo "ref rc $?"
cat gpurun_out/bench.json gpurun_out/bench_cfg5.json gpurun_out/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu launches rc $?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg5_launches.csv \
    python bench.py --config cfg5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_cfg5.log 2>&1; echo "ncu cfg5 launches rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ntt_fwd3 -s 4 -c 1 -o gpurun_out/ntt_full -f \
    python tools/ntt_once.py > gpurun_out/ncu_ntt_full.log 2>&1; echo "ncu ntt rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ks_inner -s 1 -c 1 -o gpurun_out/ks_full -f \
    python tools/ntt_once.py > gpurun_out/ncu_ks_full.log 2>&1; echo "ncu ks rc $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ks_plan -s 1 -c 1 -o gpurun_out/plan_full -f \
    python tools/plan_once.py > gpurun_out/ncu_plan_full.log 2>&1; echo "ncu plan rc $?"
echo collected
