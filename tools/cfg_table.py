"""Per-config table: one product end to end through hgm_matmul_batch (wall,
median / best of 5), the cloud phase of a lockstep batch (CUDA events, median of 5) as
matmuls/s and as a fraction of the HBM peak on SURVEY 8(d)'s op-level bytes per matmul,
and one product on the CPU oracle (reference algorithm over the CPU RNS-BFV, 1 thread;
cfg1 / cfg2 only -- the others take minutes).  Every product is checked."""
import json
import os
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2405_02238_b200 as hb  # noqa: E402
from paper_2405_02238_b200.workload import CONFIGS, batch, splitmix_matrices  # noqa: E402

OP_BYTES = {("cfg1", "enhanced"): 0.0608e9, ("cfg1", "basic"): 0.459e9, ("cfg2", "basic"): 1.2445e9,
            ("cfg2", "enhanced"): 1.2433e9, ("cfg3", "basic"): 12.347e9, ("cfg5", "enhanced"): 24.03e9,
            ("cfg5", "basic"): 24.03e9}
BATCH = {"cfg1": 1024, "cfg2": 512, "cfg3": 64, "cfg5": 4}
try:
    PEAK = float(json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"])
except Exception:
    PEAK = 6650.0
try:
    from oracle.bindings import RefLib
    HAVE_ORACLE = RefLib.available()
except Exception:
    HAVE_ORACLE = False

print(f"HBM peak {PEAK:.0f} GB/s; columns: 1-instance e2e wall ms (median / best of 5) | lockstep batch K: cloud ms, "
      f"matmuls/s, op-level GB/s, frac of peak | CPU oracle s per product (1 thread)")
for name in sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg5"]:
    m, l, n, lo, hi, pid, _, _ = CONFIGS[name]
    ctx = hb.Context(pid, 1, 0)
    A, B = splitmix_matrices(20240404, 0, m, l, n, lo, hi)
    K = BATCH[name]
    Ab, Bb = batch(20240404, 0, K, m, l, n, lo, hi)
    for algo in ("basic", "enhanced"):
        try:
            ctx.matmul_batch(A, B, algo=hb.ALGOS[algo])
        except hb.CapacityError:
            print(f"{name:5s} {algo:9s}: CapacityError (as the reference)")
            continue
        ts = []
        for _ in range(5):
            ctx.sync()
            t0 = time.perf_counter()
            C, _ = ctx.matmul_batch(A, B, algo=hb.ALGOS[algo])
            ctx.sync()
            ts.append(time.perf_counter() - t0)
        assert np.array_equal(C[0], (A @ B) % 65537)
        bt = hb.Batch(ctx, Ab, Bb, algo=hb.ALGOS[algo])
        bt.cloud()
        ms = float(np.median([bt.cloud() for _ in range(5)]))
        Cb = bt.decrypt()
        bt.free()
        assert all(np.array_equal(Cb[i], (Ab[i] @ Bb[i]) % 65537) for i in range(K))
        rate = K / ms * 1e3
        gbs = rate * OP_BYTES[(name, algo)] / 1e9
        cpu = ""
        if HAVE_ORACLE and name in ("cfg1", "cfg2"):
            t0 = time.perf_counter()
            Co, _, _, _ = RefLib.mm_oracle(A, B, param_id=pid, seed=1, counter0=0, algo=algo)
            cpu = f" | oracle {time.perf_counter() - t0:.2f} s"
            assert np.array_equal(Co, C[0])
        print(f"{name:5s} {algo:9s}: {1e3 * float(np.median(ts)):6.2f} / {1e3 * min(ts):6.2f} ms | K={K:4d}: {ms:8.2f} ms, "
              f"{rate:9.1f} matmuls/s, {gbs:7.0f} GB/s, {gbs / PEAK:5.2f}{cpu}", flush=True)
    ctx.close()
