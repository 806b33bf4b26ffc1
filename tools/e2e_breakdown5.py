"""Wall-clock split of the cfg5 end-to-end path (32 row-block products 16x128 . 128x128,
enhanced_mm at N = 32768): client encrypt, cloud phase, decrypt, and the one-call path."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import paper_2405_02238_b200 as hb  # noqa: E402
from paper_2405_02238_b200.workload import splitmix_matrices  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 32
ctx = hb.Context(1, 1, 0)
A, B = splitmix_matrices(20240505, 0, 128, 128, 128, -4, 3)
As = np.stack([A[16 * (k % 8): 16 * (k % 8) + 16] for k in range(K)])
Bs = np.stack([B for _ in range(K)])
for rep in range(3):
    ctx.sync()
    t0 = time.perf_counter()
    bt = hb.Batch(ctx, As, Bs, algo=1)
    ctx.sync()
    t1 = time.perf_counter()
    ms = bt.cloud()
    ctx.sync()
    t2 = time.perf_counter()
    C = bt.decrypt()
    t3 = time.perf_counter()
    bt.free()
    t4 = time.perf_counter()
    C2, _ = ctx.matmul_batch(As, Bs, algo=1)
    ctx.sync()
    t5 = time.perf_counter()
    print(f"rep {rep}: encrypt {1e3*(t1-t0):.1f} ms  cloud {1e3*(t2-t1):.1f} ms (device {ms:.1f})  "
          f"decrypt {1e3*(t3-t2):.1f} ms  free {1e3*(t4-t3):.1f} ms | matmul_batch {1e3*(t5-t4):.1f} ms", flush=True)
assert np.array_equal(C2[0], (As[0] @ Bs[0]) % 65537)
