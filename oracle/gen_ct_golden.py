"""TEST INFRASTRUCTURE ONLY: regenerates tests/golden/ciphertext_golden.json --
SHA-256 digests of the FINAL (pre-decrypt) ciphertext words of whole HEGMM
products, computed by the reference's own algorithms (basic_mm / enhanced_mm,
/root/reference/proj/src/algorithms.cpp:198-367, compiled in place by
oracle/ref.mk) running over the CPU RNS-BFV restatement (oracle/bfv_oracle.cpp).

These pin the GPU library's ciphertexts to the oracle bit for bit on every
BASELINE.json config (the north_star's "given identical keys and noise,
ciphertexts must be bit-exact"), where the GPU tests cannot run the oracle
themselves (it takes seconds to minutes per product and /root/reference is not
on the GPU box):

* cfg1 enhanced/basic, cfg2 basic/enhanced, cfg3 basic (N=8192, seed 2405 inputs)
* cfg5 basic/enhanced (N=32768) and the 8 row blocks A[16r:16r+16].B of the
  8-GPU decomposition (enhanced, block r encrypting from counter 2r)
* cfg4 instances 0, 1, 2047 and 4095 of the bench workload (seed 20240404,
  instance i encrypting from counter 3i, basic_mm)

Keys and noise come from the context seed (1) through the shared counter PRNG;
the digest is over the little-endian uint64 words (c0 limbs then c1 limbs).

Usage:  python oracle/gen_ct_golden.py [-j JOBS]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

OUT = os.path.join(ROOT, "tests", "golden", "ciphertext_golden.json")
GOLD_SEED = 2405      # tests/golden/reference_golden.json inputs
BENCH_SEED = 20240404  # bench.py cfg4 workload
CTX_SEED = 1


def cases():
    from paper_2405_02238_b200.workload import CONFIGS

    out = []
    for name, algos in (("cfg1", ("enhanced", "basic")), ("cfg2", ("basic", "enhanced")), ("cfg3", ("basic",)),
                        ("cfg5", ("basic", "enhanced"))):
        m, l, n, lo, hi, pid, _, _ = CONFIGS[name]
        for algo in algos:
            out.append({"case": f"{name}/{algo}", "config": name, "algo": algo, "param_id": pid,
                        "inputs": {"seed": GOLD_SEED, "index": 0, "m": m, "l": l, "n": n, "lo": lo, "hi": hi},
                        "counter0": 0})
    m, l, n, lo, hi, pid, _, _ = CONFIGS["cfg5"]
    for r in range(8):
        out.append({"case": f"cfg5/rowblock{r}", "config": "cfg5", "algo": "enhanced", "param_id": pid,
                    "inputs": {"seed": GOLD_SEED, "index": 0, "m": m, "l": l, "n": n, "lo": lo, "hi": hi,
                               "rows": [16 * r, 16 * r + 16]},
                    "counter0": 2 * r})
    m, l, n, lo, hi, pid, _, _ = CONFIGS["cfg4"]
    for i in (0, 1, 2047, 4095):
        out.append({"case": f"cfg4/instance{i}", "config": "cfg4", "algo": "basic", "param_id": pid,
                    "inputs": {"seed": BENCH_SEED, "index": i, "m": m, "l": l, "n": n, "lo": lo, "hi": hi},
                    "counter0": 3 * i})
    return out


def inputs_of(c):
    from paper_2405_02238_b200.workload import splitmix_matrices

    s = c["inputs"]
    A, B = splitmix_matrices(s["seed"], s["index"], s["m"], s["l"], s["n"], s["lo"], s["hi"])
    if "rows" in s:
        A = A[s["rows"][0]: s["rows"][1]]
    return np.ascontiguousarray(A), np.ascontiguousarray(B)


def run_case(c):
    from oracle.bindings import RefLib

    A, B = inputs_of(c)
    N = 32768 if c["param_id"] == 1 else 8192
    L = 8 if c["param_id"] == 1 else 3
    t0 = time.time()
    C, st, ct, nxt = RefLib.mm_oracle(A, B, param_id=c["param_id"], seed=CTX_SEED, counter0=c["counter0"],
                                      algo=c["algo"], words=2 * L * N)
    assert np.array_equal(C, (A @ B) % 65537), c["case"]
    rec = dict(c)
    rec.update({"ct_sha256": hashlib.sha256(ct.astype("<u8").tobytes()).hexdigest(),
                "ct_head": [int(x) for x in ct[:4]],
                "C_sha256": hashlib.sha256(np.ascontiguousarray(C, dtype=np.int64).tobytes()).hexdigest(),
                "stats": st[:12].astype(int).tolist(), "next_counter": int(nxt),
                "oracle_s": round(time.time() - t0, 1)})
    print(f"{c['case']}: {rec['oracle_s']} s", flush=True)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("-j", type=int, default=os.cpu_count() or 4)
    ap.add_argument("--only", default=None, help="substring filter on case names")
    args = ap.parse_args()
    cs = [c for c in cases() if not args.only or args.only in c["case"]]
    # slowest first (N = 32768) so the pool stays busy
    cs.sort(key=lambda c: -c["param_id"])
    with ProcessPoolExecutor(args.j) as ex:
        recs = list(ex.map(run_case, cs))
    old = {}
    if args.only and os.path.exists(OUT):
        old = {r["case"]: r for r in json.load(open(OUT))["cases"]}
    for r in recs:
        old[r["case"]] = r
    order = {c["case"]: i for i, c in enumerate(cases())}
    gold = {"generator": "oracle/gen_ct_golden.py", "ctx_seed": CTX_SEED,
            "cases": sorted(old.values(), key=lambda r: order[r["case"]])}
    with open(OUT, "w") as f:
        json.dump(gold, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
