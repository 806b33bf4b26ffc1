# ncu --set full of one launch of the kernels matching $1 inside a 64-instance cloud step
set -e
python tools/profile_step.py 64 > gpurun_out/pk_plain.txt 2>&1
SKIP=$(sed -n 's/.*skip=\([0-9]*\).*/\1/p' gpurun_out/pk_plain.txt)
ncu --set full --clock-control none --import-source on -k regex:"$1" --launch-skip-before-match 0 -s 2 -c 1 -o gpurun_out/pk_$2 python tools/profile_step.py 64 > gpurun_out/pk_$2.log 2>&1
echo done
