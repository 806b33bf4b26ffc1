#!/bin/bash
HGM_KS_SCATTER=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hegmm.py tests/test_gpu_ct_golden.py -q -x 2>&1 | tail -1
for v in 0 1 0 1; do echo -n "scatter=$v ks ms: "; HGM_KS_SCATTER=$v python -c "
import sys; sys.path.insert(0,'.')
import paper_2405_02238_b200 as hb
g=hb.Context(0,1,0); print(round(g.bench_keyswitch(2048, 10),4))"; done
bash tools/r02_ab.sh "gather|-|HGM_KS_SCATTER=0" "scatter|-|HGM_KS_SCATTER=1"
BENCH_ARGS="--config cfg5" bash tools/r02_ab.sh "cfg5-gather|-|HGM_KS_SCATTER=0" "cfg5-scatter|-|HGM_KS_SCATTER=1"
