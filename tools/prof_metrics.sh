# (the ncu pass runs under its own timeout: a 1024-instance step with these metrics outlived a 25 min gpurun limit)
# Per-kernel utilisation of one 256-instance cloud step (run under gpurun):
# DRAM throughput, integer-multiply pipe and issue activity for every launch.
set -e
python tools/profile_step.py ${K:-256} > gpurun_out/prof_plain.txt 2>&1
SKIP=$(sed -n 's/.*skip=\([0-9]*\).*/\1/p' gpurun_out/prof_plain.txt)
CNT=$(sed -n 's/.*count=\([0-9]*\).*/\1/p' gpurun_out/prof_plain.txt)
timeout ${NCU_TIMEOUT:-1200} ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size \
  --clock-control none -s $SKIP -c $CNT --csv --log-file gpurun_out/metrics.csv python tools/profile_step.py ${K:-256} > gpurun_out/ncu_metrics.log 2>&1
echo ncu_rc=$?
