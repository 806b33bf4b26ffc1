"""TEST INFRASTRUCTURE ONLY: regenerates tests/golden/reference_golden.json by
running the REFERENCE ITSELF (oracle/_ref/libhegmm_ref.so, built in place from
/root/reference/proj/src by oracle/ref.mk) on:

* the literal known-answer products of the reference's CLI tests
  (proj/tests/test_cli.cpp:75-98),
* the pinned Fig-2 diagonal plans (proj/tests/test_lintrans.cpp:110-129),
* the BASELINE.json configs 1-3 and 5 on seeded campaign inputs
  (decrypted product of SlotBackend{N/2, 65537}, per-phase op counts, and a
  digest of the full op stream: kinds, rotation offsets, cmult masks).

Usage:  python oracle/gen_golden.py   (needs /root/reference at build time only)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle.bindings import RefLib  # noqa: E402
from paper_2405_02238_b200.workload import CONFIGS, splitmix_matrices  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "reference_golden.json")
SEED = 2405


def stream_digest(hdr: np.ndarray, data: np.ndarray) -> str:
    """Canonical digest of an op stream: (kind, arg) per op and every cmult mask.
    Encrypt payloads are excluded (they are per-instance data, not the program)."""
    h = hashlib.sha256()
    off = 0
    for kind, arg, dlen in hdr.tolist():
        h.update(np.array([kind, arg], dtype=np.int64).tobytes())
        if kind == 4:
            h.update(np.ascontiguousarray(data[off:off + dlen], dtype=np.int64).tobytes())
        off += dlen
    return h.hexdigest()


def main() -> None:
    gold = {"generator": "oracle/gen_golden.py", "seed": SEED, "kats": [], "configs": {}}
    A = np.arange(1, 16, dtype=np.int64).reshape(5, 3)
    B = np.array([[1, 0, 0, 1], [0, 1, 0, 1], [0, 0, 1, 1]], dtype=np.int64)
    C, st = RefLib.mm(A, B, "basic", slots=4096)
    gold["kats"].append({"source": "proj/tests/test_cli.cpp:75-87", "algo": "basic", "A": A.tolist(),
                         "B": B.tolist(), "C": C.tolist(), "stats": st[:12].astype(int).tolist()})
    A2 = np.array([[1, 2], [3, 4]], dtype=np.int64)
    B2 = np.array([[5, 6], [7, 8]], dtype=np.int64)
    C2, st2 = RefLib.mm(A2, B2, "enhanced", slots=4096)
    gold["kats"].append({"source": "proj/tests/test_cli.cpp:89-98", "algo": "enhanced", "A": A2.tolist(),
                         "B": B2.tolist(), "C": C2.tolist(), "stats": st2[:12].astype(int).tolist()})
    gold["plans"] = [
        {"source": "proj/tests/test_lintrans.cpp:110-119", "kind": "eps", "k": 1, "m": 5, "l": 3, "n": 3,
         "order": "col", "offsets": [-10, 5], "weights": [5, 10]},
        {"source": "proj/tests/test_lintrans.cpp:121-129", "kind": "omega", "k": 1, "l": 3, "m": 3, "n": 5,
         "order": "col", "offsets": [-2, 1], "weights": [5, 10]},
    ]
    for name in ("cfg1", "cfg2", "cfg3", "cfg5"):
        m, l, n, lo, hi, pid, algos, _ = CONFIGS[name]
        slots = 16384 if pid == 1 else 4096
        A, B = splitmix_matrices(SEED, 0, m, l, n, lo, hi)
        entry = {"m": m, "l": l, "n": n, "lo": lo, "hi": hi, "slots": slots, "algos": {}}
        for algo in ("basic", "enhanced"):
            try:
                C, st = RefLib.mm(A, B, algo, slots=slots)
            except Exception as e:  # capacity rejects are part of the record
                entry["algos"][algo] = {"error": str(e)}
                continue
            hdr, data = RefLib.trace(A, B, algo, slots=slots)
            entry["algos"][algo] = {
                "C_sha256": hashlib.sha256(np.ascontiguousarray(C, dtype=np.int64).tobytes()).hexdigest(),
                "C_corner": C[:2, :2].tolist(),
                "stats": st[:12].astype(int).tolist(),
                "ops": int(hdr.shape[0]),
                "stream_sha256": stream_digest(hdr, data),
            }
        gold["configs"][name] = entry
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        json.dump(gold, f, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
