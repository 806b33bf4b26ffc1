#!/bin/bash
# A/B of library builds and environment switches on bench.py's device value
# (cfg4, no e2e / cpu baseline), two interleaved rounds.  Each case is
# "label|HGM_LIB path or -|ENV=VAL ...".
CASES=("$@")
for r in 1 2; do
  for c in "${CASES[@]}"; do
    IFS='|' read -r label lib envs <<< "$c"
    [ "$lib" = "-" ] && lib=""
    v=$(env ${lib:+HGM_LIB=$lib} $envs python bench.py --no-cpu-baseline --no-e2e $BENCH_ARGS 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read())['value'])")
    echo "$label $v"
  done
done
