#!/bin/bash
HGM_LIB=variants/lib_s1.so timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k ntt 2>&1 | tail -1
bash tools/ntt_variants.sh 2>&1 | grep -E "==|fwd=True"
args=(); for l in variants/lib_*.so; do n=$(basename $l .so); args+=("${n#lib_}|$l|"); done
bash tools/r02_ab.sh "${args[@]}"
