# SPDX-License-Identifier: Apache-2.0
# Attribution: the case draws and the Table-1 cost model restate the reference
# implementation of arXiv 2405.02238 (Apache-2.0; /root/reference/proj/src/
# costmodel.cpp:20-30, :83-106, :154-184), so that draws are bit-identical to
# run_campaign's (pinned by tests/test_campaign.py).
"""Real-HE campaign.

The reference's campaign (``run_campaign``, /root/reference/proj/src/costmodel.cpp:266-314)
draws random shapes and matrices (``run_case``, :154-208), runs every algorithm on the
cleartext ``SlotBackend`` and prices the recorded op counts with the paper's Table-1
latencies (``estimate_cost``, :32-44; weights ``costmodel.hpp:18-27``).  Here every case
runs as real BFV on the GPU (``--backend bfv-gpu``, through ``hgm_matmul_batch``), and the
report carries the MEASURED wall-clock of each encrypted product next to the cost-model
estimate for the same op counts.

Draws follow run_case exactly: per-case splitmix64 stream ``seed * 0x9e3779b97f4a7c15 +
index + 1``; m, l, n uniform in [dim_lo, dim_hi], redrawn (same stream) until every
requested algorithm fits; entries ``splitmix64() % 19 - 9``, A row-major then B.
``tests/test_campaign.py`` pins shapes and cost estimates against the reference's own
``run_campaign`` compiled in place.

    python -m paper_2405_02238_b200.campaign --cases 200 --dim-hi 64 --csv out.csv --json out.json
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from typing import Dict, List, Optional, Sequence

import numpy as np

from .workload import GOLDEN, MASK

T = 65537
ALGO_IDS = {"hegmm": 0, "hegmm-en": 1, "square-pad": 2}
# costmodel.hpp:18-27 (paper Table 1, ms per op)
TABLE1 = {"add": 0.550, "mult_cc": 20.874, "mult_cp": 4.138, "rot": 5.350, "encrypt": 5.50, "decrypt": 2.57}
OPS = ("add", "mult_cc", "mult_cp", "rot", "encrypt", "decrypt")  # stats[2k] client, [2k+1] cloud
CATEGORIES = ("m-min", "l-min", "n-min", "l-mod-m", "square")


class _Stream:
    """costmodel.cpp:20-30 splitmix64 / draw_in."""

    def __init__(self, seed: int, index: int):
        self.s = (seed * GOLDEN + index + 1) & MASK

    def next(self) -> int:
        self.s = (self.s + GOLDEN) & MASK
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        return z ^ (z >> 31)

    def draw_in(self, lo: int, hi: int) -> int:
        return lo + self.next() % (hi - lo + 1)


def classify_shape(m: int, l: int, n: int) -> List[str]:
    """costmodel.cpp:83-106."""
    p = min(m, l, n)
    out = []
    if m == p:
        out.append("m-min")
    if l == p:
        out.append("l-min")
    if n == p:
        out.append("n-min")
    if l % m == 0:
        out.append("l-mod-m")
    if m == l == n:
        out.append("square")
    return out


def fits(algo: str, m: int, l: int, n: int, slots: int, N: int) -> bool:
    """algorithms.cpp:186-196: the algorithm's segment fits the slot budget."""
    from . import CapacityError, program_info

    try:
        program_info(ALGO_IDS[algo], m, l, n, slots, N)
        return True
    except CapacityError:
        return False


def draw_case(seed: int, index: int, dim_lo: int, dim_hi: int, algos: Sequence[str], slots: int, N: int):
    """run_case's draws (costmodel.cpp:154-184): (m, l, n, A, B, resampled)."""
    st = _Stream(seed, index)
    resampled = 0
    while True:
        m, l, n = st.draw_in(dim_lo, dim_hi), st.draw_in(dim_lo, dim_hi), st.draw_in(dim_lo, dim_hi)
        if all(fits(a, m, l, n, slots, N) for a in algos):
            break
        resampled += 1
    vals = np.array([st.next() % 19 for _ in range(m * l + l * n)], dtype=np.int64) - 9
    return m, l, n, vals[: m * l].reshape(m, l), vals[m * l:].reshape(l, n), resampled


def estimate_cost(stats: Sequence[int], model: Dict[str, float] = TABLE1):
    """estimate_cost (costmodel.cpp:32-44): (client_ms, cloud_ms), same summation order."""
    out = []
    for ph in (0, 1):
        total = 0.0
        for k, op in enumerate(OPS[:4]):
            total += float(stats[2 * k + ph]) * model[op]
        for k, op in ((4, "encrypt"), (5, "decrypt")):
            total += float(stats[2 * k + ph]) * model[op]
        out.append(total)
    return out[0], out[1]


def _summarize(r: List[float]):
    if not r:
        return {"count": 0, "average": 0.0, "median": 0.0, "max": 0.0}
    r = sorted(r)
    mid = len(r) // 2
    med = r[mid] if len(r) % 2 else (r[mid - 1] + r[mid]) / 2.0
    return {"count": len(r), "average": sum(r) / len(r), "median": med, "max": r[-1]}


def _pairs(cases, algos, key):
    """summarize_pair (costmodel.cpp:232-260) over `key` (cloud_ms, or measured_ms)."""
    order = [("square-pad", "hegmm"), ("square-pad", "hegmm-en"), ("hegmm", "hegmm-en")]
    out = []
    for base, cand in order:
        if base not in algos or cand not in algos:
            continue
        overall, per = [], {c: [] for c in CATEGORIES}
        for c in cases:
            rb, rc = c["algos"].get(base), c["algos"].get(cand)
            if rb is None or rc is None or rc[key] <= 0:
                continue
            ratio = rb[key] / rc[key]
            overall.append(ratio)
            for cat in c["categories"]:
                per[cat].append(ratio)
        out.append({"baseline": base, "candidate": cand, "overall": _summarize(overall),
                    "categories": {c: _summarize(v) for c, v in per.items()}})
    return out


def run_campaign(cases: int = 500, dim_lo: int = 1, dim_hi: int = 16, seed: int = 1,
                 algos: Sequence[str] = ("hegmm", "hegmm-en", "square-pad"), backend: str = "bfv-gpu",
                 param_id: int = 0, repeats: int = 1, ctx=None, progress: bool = False) -> dict:
    """The campaign with every product encrypted on the GPU (backend "bfv-gpu") or
    only priced (backend "cost-model": op counts from the compiled program, no run)."""
    from . import Context, program_info

    own = None
    if backend == "bfv-gpu" and ctx is None:
        ctx = own = Context(param_id, seed, 0)
    slots = ctx.slot_count if ctx is not None else (4096 if param_id != 1 else 16384)
    N = ctx.N if ctx is not None else 2 * slots
    out_cases, resampled = [], 0
    ctr = 0
    try:
        for i in range(cases):
            m, l, n, A, B, rs = draw_case(seed, i, dim_lo, dim_hi, algos, slots, N)
            resampled += rs
            want = (A @ B) % T
            rec = {"case": i, "m": m, "l": l, "n": n, "categories": classify_shape(m, l, n), "algos": {}}
            for a in algos:
                if backend == "bfv-gpu":
                    ctx.matmul_batch(A, B, algo=ALGO_IDS[a], counter0=ctr)  # compiles the shape's program
                    ctr += 8
                    best = None
                    for _ in range(max(1, repeats)):
                        ctx.sync()
                        t0 = time.perf_counter()
                        C, st = ctx.matmul_batch(A, B, algo=ALGO_IDS[a], counter0=ctr)
                        dt = (time.perf_counter() - t0) * 1e3
                        ctr += 8
                        best = dt if best is None else min(best, dt)
                    exact = bool(np.array_equal(C[0], want))
                else:
                    st, _ = program_info(ALGO_IDS[a], m, l, n, slots, N)
                    best, exact = None, None
                stats = [int(x) for x in st[:12]]
                client, cloud = estimate_cost(stats)
                rec["algos"][a] = {"exact": exact, "stats": stats, "client_ms": client, "cloud_ms": cloud,
                                   "total_ms": client + cloud, "measured_ms": best}
            out_cases.append(rec)
            if progress and (i + 1) % 50 == 0:
                print(f"{i + 1}/{cases}", file=sys.stderr, flush=True)
    finally:
        if own is not None:
            own.close()
    res = {"config": {"cases": cases, "dim_lo": dim_lo, "dim_hi": dim_hi, "seed": seed, "slot_count": slots,
                      "algos": list(algos), "plaintext_modulus": T, "backend": backend, "param_id": param_id,
                      "N": N},
           "resampled": resampled, "cases": out_cases,
           "summaries": _pairs(out_cases, algos, "cloud_ms")}
    if backend == "bfv-gpu":
        res["measured_summaries"] = _pairs(out_cases, algos, "measured_ms")
    return res


def emit_csv(res: dict, f) -> None:
    """emit_csv's columns (costmodel.cpp:316-341) plus measured_ms."""
    f.write("case,m,l,n,categories,algo,exact,add_client,add_cloud,mult_cc_client,mult_cc_cloud,"
            "mult_cp_client,mult_cp_cloud,rot_client,rot_cloud,encrypt_client,encrypt_cloud,decrypt_client,"
            "decrypt_cloud,client_ms,cloud_ms,total_ms,measured_ms\n")
    for c in res["cases"]:
        for a, r in c["algos"].items():
            ex = "" if r["exact"] is None else str(int(r["exact"]))
            meas = "" if r["measured_ms"] is None else f"{r['measured_ms']:.6f}"
            f.write(f"{c['case']},{c['m']},{c['l']},{c['n']},{';'.join(c['categories'])},{a},{ex},"
                    + ",".join(str(x) for x in r["stats"])
                    + f",{r['client_ms']:.6f},{r['cloud_ms']:.6f},{r['total_ms']:.6f},{meas}\n")


def main(argv: Optional[Sequence[str]] = None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--cases", type=int, default=500)
    ap.add_argument("--dim-lo", type=int, default=1)
    ap.add_argument("--dim-hi", type=int, default=16)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--algos", default="hegmm,hegmm-en,square-pad")
    ap.add_argument("--backend", choices=("bfv-gpu", "cost-model"), default="bfv-gpu")
    ap.add_argument("--param", type=int, default=0)
    ap.add_argument("--repeats", type=int, default=1)
    ap.add_argument("--csv")
    ap.add_argument("--json")
    a = ap.parse_args(argv)
    res = run_campaign(a.cases, a.dim_lo, a.dim_hi, a.seed, a.algos.split(","), a.backend, a.param, a.repeats,
                       progress=True)
    if a.csv:
        with open(a.csv, "w") as f:
            emit_csv(res, f)
    if a.json:
        with open(a.json, "w") as f:
            json.dump(res, f, indent=1)
    exact = [r["exact"] for c in res["cases"] for r in c["algos"].values() if r["exact"] is not None]
    summ = {"cases": a.cases, "resampled": res["resampled"], "all_exact": all(exact) if exact else None,
            "cost_model": [(s["baseline"], s["candidate"], round(s["overall"]["average"], 4))
                           for s in res["summaries"]]}
    if "measured_summaries" in res:
        summ["measured"] = [(s["baseline"], s["candidate"], round(s["overall"]["average"], 4))
                            for s in res["measured_summaries"]]
        tot = {alg: sum(c["algos"][alg]["measured_ms"] for c in res["cases"]) for alg in res["config"]["algos"]}
        summ["measured_total_ms"] = {k: round(v, 2) for k, v in tot.items()}
    print(json.dumps(summ))
    return 0


if __name__ == "__main__":
    sys.exit(main())
