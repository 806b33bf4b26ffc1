#!/bin/bash
# prescaled masked keys (P^-1 folded into the Q limbs' masks, HGM_PRESCALE): GPU tests, then A/B
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/exp3_tests.log 2>&1
echo "tests rc $?"; tail -3 gpurun_out/exp3_tests.log
bash tools/r02_ab.sh "pre0|-|HGM_PRESCALE=0" "pre1|-|HGM_PRESCALE=1"
BENCH_ARGS="--config cfg5" bash tools/r02_ab.sh "c5pre0|-|HGM_PRESCALE=0" "c5pre1|-|HGM_PRESCALE=1"
