#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_configs.py tests/test_gpu_ct_golden.py -q -x 2>&1 | tail -2
BENCH_ARGS="--config cfg5" bash tools/r02_ab.sh "cfg5-cur|-|" "cfg5-lcgen|-|HGM_LC_MASKED=0" "cfg5-noadd|variants/lib_noadd.so|"
bash tools/r02_ab.sh "cfg4-cur|-|" "cfg4-lcgen|-|HGM_LC_MASKED=0"
