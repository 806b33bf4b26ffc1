# SPDX-License-Identifier: Apache-2.0
# Attribution: the splitmix64 draws restate the reference implementation of
# arXiv 2405.02238 (Apache-2.0; /root/reference/proj/src/costmodel.cpp:20-26, :158-184).
"""Seeded synthetic HEGMM workloads (BASELINE.json configs).

Entries are drawn exactly as the reference's seeded campaign draws them
(/root/reference/proj/src/costmodel.cpp:20-26 splitmix64; per-instance stream
seed*0x9e3779b97f4a7c15 + index + 1 at :158; A filled row-major, then B,
:172-184), with entry = lo + splitmix64() % (hi - lo + 1).
"""
from __future__ import annotations

import numpy as np

MASK = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15

# name -> (m, l, n, lo, hi, param_id, algos, instances)
CONFIGS = {
    "cfg1": (8, 16, 4, -8, 7, 0, ("enhanced", "basic"), 1),
    "cfg2": (64, 64, 64, -8, 7, 0, ("basic", "enhanced"), 1),
    "cfg3": (32, 128, 16, -4, 3, 0, ("basic",), 1),
    "cfg4": (64, 64, 64, -8, 7, 0, ("basic", "enhanced"), 4096),
    "cfg5": (128, 128, 128, -4, 3, 1, ("enhanced", "basic"), 1),
}


def splitmix_matrices(seed: int, index: int, m: int, l: int, n: int, lo: int, hi: int):
    """One instance's (A, B), bit-identical to the reference campaign's draw."""
    state = (seed * GOLDEN + index + 1) & MASK
    span = hi - lo + 1
    out = np.empty(m * l + l * n, dtype=np.int64)
    for k in range(out.size):
        state = (state + GOLDEN) & MASK
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        z ^= z >> 31
        out[k] = lo + z % span
    return out[: m * l].reshape(m, l), out[m * l:].reshape(l, n)


def batch(seed: int, first: int, count: int, m: int, l: int, n: int, lo: int, hi: int):
    """Instances first..first+count-1 stacked as (count, m, l), (count, l, n);
    the same draws as splitmix_matrices, vectorised (uint64 arithmetic wraps)."""
    total = m * l + l * n
    g = np.uint64(GOLDEN)
    with np.errstate(over="ignore"):
        base = (np.uint64(seed % (1 << 64)) * g + np.arange(first, first + count, dtype=np.uint64)
                + np.uint64(1))
        z = base[:, None] + g * np.arange(1, total + 1, dtype=np.uint64)[None, :]
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    vals = (np.int64(lo) + (z % np.uint64(hi - lo + 1)).astype(np.int64))
    A = np.ascontiguousarray(vals[:, : m * l].reshape(count, m, l))
    B = np.ascontiguousarray(vals[:, m * l:].reshape(count, l, n))
    return A, B
