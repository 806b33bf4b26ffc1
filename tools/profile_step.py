"""One warm-up cloud step, then one profiled cloud step of the bench workload
(smaller batch).  Prints the launch counts so ncu can skip the warm-up:
  python tools/profile_step.py K            -> prints "skip=<n> count=<n>"
  ncu -s <skip> -c <count> ... python tools/profile_step.py K
"""
import sys

sys.path.insert(0, ".")
import paper_2405_02238_b200 as hb  # noqa: E402
from paper_2405_02238_b200.workload import batch  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 256
algo = int(sys.argv[2]) if len(sys.argv) > 2 else 0
ctx = hb.Context(0, 1, 0)
A, B = batch(20240404, 0, K, 64, 64, 64, -8, 7)
bt = hb.Batch(ctx, A, B, algo=algo)
bt.cloud()
ctx.sync()
l0 = ctx.launch_count()
ms = bt.cloud()
ctx.sync()
l1 = ctx.launch_count()
print(f"skip={l0} count={l1 - l0} cloud_ms={ms:.3f} rate={K / ms * 1e3:.1f}/s", flush=True)
