import sys
sys.path.insert(0, '.')
import paper_2405_02238_b200 as hb
for pid, lb in ((0, 131072), (1, 524288)):
    g = hb.Context(pid, 1, 0)
    limbs = 148 * 8 if pid == 0 else 148 * 2
    for fwd in (True, False):
        ms = g.bench_ntt(limbs, 20, fwd)
        print(f"pid={pid} fwd={fwd} limbs={limbs}: {limbs*lb/ms/1e6:.1f} GB/s ({ms*1e3/limbs:.1f} ns/limb)", flush=True)
    g.close()
