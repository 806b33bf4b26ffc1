"""Invariant-noise budget (bits, oracle measure) left in each config's product ciphertext."""
import sys

sys.path.insert(0, ".")
import paper_2405_02238_b200 as hb  # noqa: E402
from oracle.bindings import Oracle  # noqa: E402
from paper_2405_02238_b200.workload import CONFIGS, splitmix_matrices  # noqa: E402

for name, algo in [("cfg1", "enhanced"), ("cfg1", "basic"), ("cfg2", "basic"), ("cfg2", "enhanced"),
                   ("cfg3", "basic"), ("cfg5", "basic"), ("cfg5", "enhanced")]:
    m, l, n, lo, hi, pid, _, _ = CONFIGS[name]
    A, B = splitmix_matrices(20240404, 0, m, l, n, lo, hi)
    ctx = hb.Context(pid, 1, 0)
    C, words = ctx.matmul_batch(A, B, algo=hb.ALGOS[algo], export=True)
    print(f"{name} {algo}: {Oracle(pid, 1).noise_budget(words[0]):.1f} bits left", flush=True)
    ctx.close()
