#!/bin/bash
# tw-cache fill loop rolled (no trip-count division, data loads ahead of the cp.async wait) vs unrolled
timeout 600 python -m pytest tests -m gpu -x -q -k "parity or ntt or configs" > gpurun_out/exp4_tests.log 2>&1
echo "tests rc $?"; tail -2 gpurun_out/exp4_tests.log
for r in 1 2; do
  for v in unrolled main; do
    lib=variants/lib_$v.so; [ $v = main ] && lib=""
    out=$(env ${lib:+HGM_LIB=$lib} timeout 300 python bench.py --no-cpu-baseline --no-e2e $BENCH_ARGS 2>/dev/null)
    echo "$v $(echo "$out" | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print(d['value'], 'fwd', r['achieved'], 'inv_frac', r['inverse_frac'])")"
  done
done
