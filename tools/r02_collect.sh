#!/bin/bash
# Round-2 evidence (run under gpurun, one GPU): GPU tests, both bench lines
# (cfg4 default + cfg5), the reference arm, the ncu launch list of the bench
# command and ncu --set full captures of the forward NTT and k_ks_inner launches
# bench.py's roofline times.
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
if [ -z "$SKIP_TESTS" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc $?" >> gpurun_out/gputest.log
  tail -3 gpurun_out/gputest.log
fi
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
timeout 600 python bench.py --config cfg5 --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "cfg5 rc $?"
cat gpurun_out/bench.json gpurun_out/bench_cfg5.json
if [ -n "$REF_ARM" ]; then
  timeout 600 python bench.py --impl reference --steps 1 --warmup 3 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
fi
if [ -n "$NCU" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv \
      python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1; echo "ncu launches rc $?"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ntt_fwd3 -s 4 -c 1 -o gpurun_out/ntt_full -f \
      python tools/ntt_once.py > gpurun_out/ncu_ntt_full.log 2>&1; echo "ncu ntt rc $?"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ks_inner -s 1 -c 1 -o gpurun_out/ks_full -f \
      python tools/ntt_once.py > gpurun_out/ncu_ks_full.log 2>&1; echo "ncu ks rc $?"
fi
echo collected
