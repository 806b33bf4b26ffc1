"""Wall time of one product per config through hgm_matmul_batch (after a warm-up
run that generates keys and masks): median and best of 5."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2405_02238_b200 as hb  # noqa: E402
from paper_2405_02238_b200.workload import CONFIGS, splitmix_matrices  # noqa: E402

for name in sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg5"]:
    m, l, n, lo, hi, pid, _, _ = CONFIGS[name]
    ctx = hb.Context(pid, 1, 0)
    A, B = splitmix_matrices(20240404, 0, m, l, n, lo, hi)
    for algo in ("basic", "enhanced"):
        try:
            ctx.matmul_batch(A, B, algo=hb.ALGOS[algo])
        except hb.CapacityError:
            print(f"{name} {algo}: CapacityError")
            continue
        ts = []
        for _ in range(5):
            ctx.sync()
            t0 = time.perf_counter()
            C, _ = ctx.matmul_batch(A, B, algo=hb.ALGOS[algo])
            ctx.sync()
            ts.append(time.perf_counter() - t0)
        ok = np.array_equal(C[0], (A @ B) % 65537)
        print(f"{name} {algo}: median {1e3 * float(np.median(ts)):.1f} ms, best {1e3 * min(ts):.1f} ms per product "
              f"(1 instance, wall), exact={ok}", flush=True)
    ctx.close()
