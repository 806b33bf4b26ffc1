"""The paper's only absolute timing (Table 4): a 100x100 . 100x100
product, blocked P1 (50/50 halves) and P2 (64/36), HEGMM and HEGMM-En.  The
paper: Pyfhel BFV N=2^12 on a 10-core Xeon, 39.12 / 39.15 s (P1), 26.17 /
26.23 s (P2).  Here: BFV N=8192 on one B200, end to end (encrypt, every block
product, decrypt, accumulate).  Prints one JSON line per case."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2405_02238_b200 as hb  # noqa: E402

ctx = hb.Context(0, 1, 0)
rng = np.random.default_rng(2024)
A = rng.integers(-9, 10, (100, 100))
B = rng.integers(-9, 10, (100, 100))
for split, parts in (("P1", [50, 50]), ("P2", [64, 36])):
    for algo, name in ((0, "HEGMM"), (1, "HEGMM-En")):
        ctx.blocked_mm(A, B, parts, parts, parts, algo=algo)  # warm keys, masks, programs
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            C, log = ctx.blocked_mm(A, B, parts, parts, parts, algo=algo)
            ts.append(time.perf_counter() - t0)
        assert np.array_equal(C, (A @ B) % 65537)
        paper = {("P1", 0): 39.12, ("P1", 1): 39.15, ("P2", 0): 26.17, ("P2", 1): 26.23}[(split, algo)]
        print(json.dumps({"case": f"100x100 {split} {name}", "seconds_median": round(float(np.median(ts)), 4),
                          "seconds_best": round(min(ts), 4), "paper_cpu_seconds": paper,
                          "blocks": int(len(log)), "fallbacks": int(log[:, 1].sum())}), flush=True)
