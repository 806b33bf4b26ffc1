import sys
sys.path.insert(0, '.')
import paper_2405_02238_b200 as hb
g = hb.Context(0, 1, 0)
g.bench_ntt(148 * 8, 2, True)
g.bench_ntt(148 * 8, 2, False)
print("ok")
