#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ct_golden.py tests/test_gpu_configs.py tests/test_gpu_hegmm.py -q -x 2>&1 | tail -2
HGM_FUSED_KS=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
HGM_NTT_CLUSTER=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ct_golden.py -q -x -k "1 or cfg5" 2>&1 | tail -1
BENCH_ARGS="--config cfg5" bash tools/r02_ab.sh "cfg5-head|variants/lib_a_head.so|" "cfg5-new|-|"
bash tools/r02_ab.sh "cfg4-head|variants/lib_a_head.so|" "cfg4-new|-|"
