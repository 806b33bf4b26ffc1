#!/bin/bash
# bench.py (device value only) for every variants/lib_*.so, twice, interleaved
for r in 1 2; do
  for l in variants/lib_*.so; do
    echo -n "$l "
    HGM_LIB=$l python bench.py --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; print(json.loads(sys.stdin.read())['value'])"
  done
done
