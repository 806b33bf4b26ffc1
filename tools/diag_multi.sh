#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "ntt" 2>&1 | tail -1
for m in 1 2 1 2; do echo -n "multi=$m "; HGM_NTT_MULTI=$m python tools/ntt_bench.py 2>&1 | grep "pid=0 fwd=True"; done
bash tools/r02_ab.sh "multi1|-|HGM_NTT_MULTI=1" "multi2|-|HGM_NTT_MULTI=2"
