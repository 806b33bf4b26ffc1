"""The k_ks_plan launch bench.py's roofline times (for ncu captures)."""
import sys
sys.path.insert(0, '.')
import paper_2405_02238_b200 as hb
pid = int(sys.argv[1]) if len(sys.argv) > 1 else 0
g = hb.Context(pid, 1, 0)
args = (128, 63, 2, 16) if g.N == 8192 else (16, 16, 2, 16)
print("ms", g.bench_keyswitch_plan(*args, 2))
