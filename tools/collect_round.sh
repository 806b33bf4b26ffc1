#!/bin/bash
# Everything profiles/ is refreshed from (run under gpurun, one GPU):
#   bench line (+ reference arm), the ncu launch list of the bench command itself,
#   ncu --set full of the forward NTT's roofline launch, per-kernel metrics of a
#   1024-instance cloud step.  Then run tools/refresh_profiles.sh here.
set -e
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
python tools/ntt_once.py > gpurun_out/ntt_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_ntt_fwd -s 3 -c 1 -o gpurun_out/ntt_full \
    python tools/ntt_once.py > gpurun_out/ncu_ntt_full.log 2>&1
K=1024 bash tools/prof_launches.sh > /dev/null
K=1024 bash tools/prof_metrics.sh
echo collected
