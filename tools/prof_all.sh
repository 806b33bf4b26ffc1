# Collects the round's evidence on one B200 (run under gpurun):
#   bench line, launch list of one cloud step (per-kernel shares), and one
#   ncu --set full capture of the forward NTT in the bench's roofline launch.
set -e
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
bash tools/prof_launches.sh
python tools/ntt_once.py > gpurun_out/ntt_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_ntt_fwd -s 3 -c 1 -o gpurun_out/ntt_full python tools/ntt_once.py > gpurun_out/ncu_ntt_full.log 2>&1
echo done
