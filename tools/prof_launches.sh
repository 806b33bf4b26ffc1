set -e
python tools/profile_step.py ${K:-256} > gpurun_out/prof_plain.txt 2>&1
cat gpurun_out/prof_plain.txt
SKIP=$(sed -n 's/.*skip=\([0-9]*\).*/\1/p' gpurun_out/prof_plain.txt)
CNT=$(sed -n 's/.*count=\([0-9]*\).*/\1/p' gpurun_out/prof_plain.txt)
ncu --metrics gpu__time_duration.sum --clock-control none -s $SKIP -c $CNT --csv --log-file gpurun_out/launches.csv python tools/profile_step.py ${K:-256} > gpurun_out/ncu_launch.log 2>&1
echo ncu_rc=$?
