#!/bin/bash
# A/B of the variants/lib_*.so builds: parity smoke, NTT GB/s, bench device value
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "ntt or rot" 2>&1 | tail -1
bash tools/ntt_variants.sh
args=()
for l in variants/lib_*.so; do n=$(basename $l .so); args+=("${n#lib_}|$l|"); done
bash tools/r02_ab.sh "${args[@]}"
