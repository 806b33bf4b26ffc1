#!/bin/bash
# A/B of the table-reduced last stage (HGM_LAST_TAB) and the one-reduction k_ks_plan
# (HGM_PLAN_WIDE): parity tests on the main build first, then bench.py's device value,
# forward NTT GB/s, FinishIO-free k_ks_plan ms per variant, two interleaved rounds.
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or configs or hegmm or ntt" > gpurun_out/exp2_tests.log 2>&1
echo "tests rc $?"; tail -2 gpurun_out/exp2_tests.log
for r in 1 2; do
  for v in base tab wide tab2 main; do
    lib=variants/lib_$v.so; [ $v = main ] && lib=""
    out=$(env ${lib:+HGM_LIB=$lib} timeout 300 python bench.py --no-cpu-baseline --no-e2e $BENCH_ARGS 2>/dev/null)
    echo "$v $(echo "$out" | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(d['value'], 'fwd', r['achieved'], 'inv_frac', r['inverse_frac'], 'plan_ms', r['keyswitch_plan']['ms_per_launch'], 'ks_ms', r['keyswitch']['ms_per_launch'])")"
  done
done
