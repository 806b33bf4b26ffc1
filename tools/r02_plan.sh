#!/bin/bash
# A/B of the masked-key plan sums (HGM_KS_PLAN): parity tests first, then bench.py device value.
timeout 900 python -m pytest tests/test_gpu_hegmm.py tests/test_gpu_ct_golden.py tests/test_gpu_configs.py tests/test_gpu_widen.py -m gpu -x -q > gpurun_out/plan_test.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/plan_test.log
for v in 1 0; do
  HGM_KS_PLAN=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/plan_bench_$v.json 2> gpurun_out/plan_bench_$v.err; echo "bench plan=$v rc $?"
  python -c "import json;d=json.load(open('gpurun_out/plan_bench_$v.json'));print('plan=$v', d['value'], d['ms_per_step'])"
done
for t in 8 32; do
  HGM_PLAN_TILE=$t timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/plan_bench_t$t.json 2> gpurun_out/plan_bench_t$t.err
  python -c "import json;d=json.load(open('gpurun_out/plan_bench_t$t.json'));print('tile=$t', d['value'], d['ms_per_step'])"
done
HGM_KS_PLAN=1 timeout 600 python bench.py --config cfg5 --no-cpu-baseline --no-e2e > gpurun_out/plan_cfg5_1.json 2> gpurun_out/plan_cfg5_1.err
HGM_KS_PLAN=0 timeout 600 python bench.py --config cfg5 --no-cpu-baseline --no-e2e > gpurun_out/plan_cfg5_0.json 2> gpurun_out/plan_cfg5_0.err
python -c "
import json
for v in (1,0):
    d=json.load(open('gpurun_out/plan_cfg5_%d.json'%v)); print('cfg5 plan=%d'%v, d['value'])"
