#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_hegmm.py tests/test_gpu_ct_golden.py tests/test_gpu_widen.py -m gpu -x -q > gpurun_out/plan_test.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/plan_test.log
for t in ${TILES:-16 8 32}; do
  HGM_PLAN_TILE=$t timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/plan_bench_t$t.json 2> gpurun_out/plan_bench_t$t.err
  python -c "import json;d=json.load(open('gpurun_out/plan_bench_t$t.json'));print('tile=$t', d['value'], d['ms_per_step'])"
done
timeout 600 python bench.py --config cfg5 --no-cpu-baseline --no-e2e > gpurun_out/plan_cfg5_1.json 2> gpurun_out/plan_cfg5_1.err
python -c "
import json
d=json.load(open('gpurun_out/plan_cfg5_1.json')); print('cfg5', d['value'])"
