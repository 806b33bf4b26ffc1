#!/bin/bash
# Times the N=8192 forward/inverse NTT of every variants/lib_*.so (tools/build_variant.sh)
for l in variants/lib_*.so; do
  echo "== $l"
  HGM_LIB=$l python - <<'PY'
import sys
sys.path.insert(0, '.')
import paper_2405_02238_b200 as hb
g = hb.Context(0, 1, 0)
for rep in range(2):
    for fwd in (True, False):
        ms = g.bench_ntt(4736, 20, fwd)
        print(f"fwd={fwd}: {4736*131072/ms/1e6:.1f} GB/s", flush=True)
g.close()
PY
done
