"""Quick performance probe (not the bench contract): NTT GB/s and batched HEGMM rate."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
import paper_2405_02238_b200 as hb
from paper_2405_02238_b200.workload import batch

g = hb.Context(0, 1, 0)
for limbs in (148 * 4, 148 * 16):
    for fwd in (True, False):
        ms = g.bench_ntt(limbs, 20, fwd)
        print(f"NTT N=8192 fwd={fwd} limbs={limbs}: {ms*1e3/limbs:.2f} us/limb-batch-share, "
              f"{limbs*131072/ms/1e6:.1f} GB/s", flush=True)
for K in (1, 16, 64, 256):
    A, B = batch(1, 0, K, 64, 64, 64, -8, 7)
    g.matmul_batch(A, B, algo=0)  # warm (keys, masks)
    t = time.time(); C, _ = g.matmul_batch(A, B, algo=0); dt = time.time() - t
    ok = all(np.array_equal(C[i], (A[i] @ B[i]) % 65537) for i in range(min(K, 4)))
    print(f"cfg2 basic K={K}: {dt*1e3:.1f} ms  -> {K/dt:.1f} matmul/s  ok={ok}  launches={g.launch_count()}", flush=True)
