"""Wall-clock split of the end-to-end path for the bench workload (4096 x 64^3):
client encrypt (pack + H2D + encrypt), cloud phase, decrypt (decrypt + D2H + unpack)."""
import sys
import time

sys.path.insert(0, ".")
import paper_2405_02238_b200 as hb  # noqa: E402
from paper_2405_02238_b200.workload import batch  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
ctx = hb.Context(0, 1, 0)
A, B = batch(20240404, 0, K, 64, 64, 64, -8, 7)
for rep in range(2):
    ctx.sync()
    t0 = time.perf_counter()
    bt = hb.Batch(ctx, A, B, algo=0)
    ctx.sync()
    t1 = time.perf_counter()
    bt.cloud()
    ctx.sync()
    t2 = time.perf_counter()
    C = bt.decrypt()
    t3 = time.perf_counter()
    bt.free()
    t4 = time.perf_counter()
    C2, _ = ctx.matmul_batch(A, B, algo=0)
    ctx.sync()
    t5 = time.perf_counter()
    print(f"rep {rep}: encrypt {1e3*(t1-t0):.1f} ms  cloud {1e3*(t2-t1):.1f} ms  decrypt {1e3*(t3-t2):.1f} ms  "
          f"free {1e3*(t4-t3):.1f} ms | matmul_batch {1e3*(t5-t4):.1f} ms", flush=True)
