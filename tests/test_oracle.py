"""CPU: pins the BFV oracle (oracle/bfv_oracle.cpp) before it is trusted.

* its NTT against the definition  out[k] = sum_j a_j psi^(j (2 brv(k) + 1));
* its primitives against plain modular arithmetic on the slots, including
  the reference's left-rotation semantics (backend.cpp:185-197, row-wide);
* the reference's own algorithms running on it against the reference's
  golden vectors (test_cli.cpp KATs, seeded config outputs) and against the
  reference SlotBackend{N/2, 65537} on random shapes."""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2405_02238_b200.workload import CONFIGS, splitmix_matrices

T = 65537
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def brv(x, bits):
    return int(f"{x:0{bits}b}"[::-1], 2)


def test_ntt_matches_definition(oracle_factory):
    o = oracle_factory(2)
    N, logN = o.N, o.N.bit_length() - 1
    rng = np.random.default_rng(1)
    for prime in (0, len(o.primes) - 1, -1):
        q = T if prime < 0 else o.primes[prime]
        a = [int(x) % q for x in rng.integers(0, 2**62, N)]
        out = o.ntt(np.array(a, dtype=np.uint64), prime)
        # psi: the primitive 2N-th root the oracle uses is out[0] of X = (0, 1, 0, ...)
        x = np.zeros(N, dtype=np.uint64)
        x[1] = 1
        psi = int(o.ntt(x, prime)[0])
        assert pow(psi, N, q) == q - 1
        for k in rng.integers(0, N, 6):
            e = 2 * brv(int(k), logN) + 1
            want = sum(aj * pow(psi, j * e, q) for j, aj in enumerate(a)) % q
            assert int(out[k]) == want
        assert np.array_equal(o.ntt(out, prime, forward=False), np.array(a, dtype=np.uint64))


def test_primitives_decrypt_correctly(oracle_factory):
    o = oracle_factory(2)
    H = o.N // 2
    rng = np.random.default_rng(2)
    S = 200
    a = rng.integers(-8, 8, S)
    b = rng.integers(-8, 8, S)
    ca, cb = o.encrypt(a, 0), o.encrypt(b, 1)
    assert np.array_equal(o.decrypt(ca, S), a % T)
    assert np.array_equal(o.decrypt(o.add(ca, cb), S), (a + b) % T)
    m = rng.integers(0, 2, S)
    assert np.array_equal(o.decrypt(o.cmult(ca, m), S), (a * m) % T)
    assert np.array_equal(o.decrypt(o.mult(ca, cb), S), (a * b) % T)
    full = np.zeros(H, dtype=np.int64)
    full[:S] = a
    for z in (1, -1, 17, H - 1, 0, H + 3):
        assert np.array_equal(o.decrypt(o.rot(ca, z), S), np.roll(full, -z)[:S] % T)
    # the rotation composes additively over the row (test_backend.cpp:102-115, row-wide)
    assert np.array_equal(o.decrypt(o.rot(o.rot(ca, 5), 7), S), o.decrypt(o.rot(ca, 12), S))


def test_noise_budget_after_mult(oracle_factory):
    o = oracle_factory(0)
    rng = np.random.default_rng(3)
    a, b = rng.integers(-8, 8, 64), rng.integers(-8, 8, 64)
    p = o.mult(o.encrypt(a, 0), o.encrypt(b, 1))
    assert o.noise_budget(p) > 20  # fixed-point measure saturates near 61 bits


def test_pending_products(oracle_factory):
    """he_mult is a pending product; he_add sums pending tensors (one
    scale-and-round + relinearisation at materialisation, bfv_oracle.cpp XCt)."""
    o = oracle_factory(2)
    rng = np.random.default_rng(4)
    S = 300
    v = [rng.integers(-8, 8, S) for _ in range(5)]
    c = [o.encrypt(x, i) for i, x in enumerate(v)]
    p01 = o.mult_pending(c[0], c[1])
    # a lone pending product materialises to the eager product, bit for bit
    assert np.array_equal(o.plain(p01), o.mult(c[0], c[1]))
    # plain + plain is the plain add
    assert np.array_equal(o.plain(o.add_any((c[0], False), (c[1], False))), o.add(c[0], c[1]))
    # zero + products + plain addend, in any association
    s1 = o.add_any(o.add_any((c[4], False), p01), o.mult_pending(c[2], c[3]))
    s2 = o.add_any(p01, o.add_any(o.mult_pending(c[2], c[3]), (c[4], False)))
    assert s1[1] and s2[1]
    m1 = o.plain(s1)
    assert np.array_equal(m1, o.plain(s2))
    assert np.array_equal(o.decrypt(m1, S), (v[0] * v[1] + v[2] * v[3] + v[4]) % T)
    # one rounding instead of two: at least the eager sum's noise budget
    eager = o.add(o.add(c[4], o.mult(c[0], c[1])), o.mult(c[2], c[3]))
    assert np.array_equal(o.decrypt(eager, S), o.decrypt(m1, S))
    assert o.noise_budget(m1) >= o.noise_budget(eager) - 1.0


def test_pending_key_switches(oracle_factory):
    """he_rot is a pending key switch (bfv_oracle.cpp XCt part A): masked sums of
    rotations are moded down once; a lone rotation materialises to the eager one."""
    o = oracle_factory(2)
    H = o.N // 2
    rng = np.random.default_rng(5)
    S = 200
    a, b = rng.integers(-8, 8, S), rng.integers(-8, 8, S)
    ca, cb = o.encrypt(a, 0), o.encrypt(b, 1)
    full = np.zeros(H, dtype=np.int64)
    full[:S] = a
    r1, r5 = o.rot_x(ca, 1), o.rot_x(ca, 5)
    assert r1[1] == 2 and o.rot_x(ca, 0)[1] == 0
    assert np.array_equal(o.plain(r1), o.rot(ca, 1))
    m1, m2 = rng.integers(0, 2, S), rng.integers(0, 2, S)
    s = o.add_any(o.cmult_x(r1, m1), o.cmult_x(r5, m2))
    want = (np.roll(full, -1)[:S] * m1 + np.roll(full, -5)[:S] * m2) % T
    assert np.array_equal(o.decrypt(o.plain(s), S), want)
    # masks distribute exactly over pending sums
    assert np.array_equal(o.plain(o.cmult_x(o.add_any(r1, r5), m1)),
                          o.plain(o.add_any(o.cmult_x(r1, m1), o.cmult_x(r5, m1))))
    # all three parts at once: plain + pending key switch + pending product
    mix = o.add_any(o.add_any((cb, 0), r1), o.mult_pending(ca, cb))
    assert mix[1] == 3
    assert np.array_equal(o.decrypt(o.plain(mix), S), (b + np.roll(full, -1)[:S] + a * b) % T)
    # masking a value with a pending product materialises it first
    mm = o.cmult_x(mix, m1)
    assert mm[1] == 0
    assert np.array_equal(o.decrypt(o.plain(mm), S), ((b + np.roll(full, -1)[:S] + a * b) * m1) % T)


def test_error_conventions(oracle_factory):
    from oracle.bindings import OracleError

    o = oracle_factory(2)
    with pytest.raises(OracleError, match="DimensionError"):
        o.encrypt(np.zeros(0, np.int64), 0)
    with pytest.raises(OracleError, match="CapacityError"):
        o.encrypt(np.zeros(o.N // 2 + 1, np.int64), 0)


def test_reference_kats_through_oracle(ref):
    for kat in GOLD["kats"]:
        A, B = np.array(kat["A"]), np.array(kat["B"])
        C, st, _, _ = ref.mm_oracle(A, B, param_id=2, algo=kat["algo"])
        assert C.tolist() == kat["C"], kat["source"]
        assert st[:12].astype(int).tolist() == kat["stats"]


def test_cfg1_through_oracle_matches_golden(ref):
    g = GOLD["configs"]["cfg1"]
    A, B = splitmix_matrices(GOLD["seed"], 0, g["m"], g["l"], g["n"], g["lo"], g["hi"])
    for algo in ("enhanced", "basic"):
        C, st, _, _ = ref.mm_oracle(A, B, param_id=0, algo=algo)
        rec = g["algos"][algo]
        assert hashlib.sha256(C.astype(np.int64).tobytes()).hexdigest() == rec["C_sha256"]
        assert st[:12].astype(int).tolist() == rec["stats"]


def test_random_shapes_oracle_vs_slotbackend(ref):
    rng = np.random.default_rng(4)
    for _ in range(6):
        m, l, n = (int(x) for x in rng.integers(1, 9, 3))
        A = rng.integers(-9, 10, (m, l))
        B = rng.integers(-9, 10, (l, n))
        for algo in ("basic", "enhanced"):
            C, _, _, _ = ref.mm_oracle(A, B, param_id=2, algo=algo)
            Cref, _ = ref.mm(A, B, algo, slots=2048)
            assert np.array_equal(C, Cref), (m, l, n, algo)


def test_ciphertext_golden_reproduces_on_cpu(ref):
    """The committed whole-product ciphertext digests (tests/golden/
    ciphertext_golden.json, pinned by the GPU tests) are what the reference's
    algorithms over the oracle produce -- checked here on the cheap cases."""
    import hashlib
    import json

    from paper_2405_02238_b200.workload import splitmix_matrices

    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ciphertext_golden.json")))
    cases = {r["case"]: r for r in gold["cases"]}
    assert len(cases) == 19
    for name in ("cfg1/enhanced", "cfg1/basic"):
        rec = cases[name]
        s = rec["inputs"]
        A, B = splitmix_matrices(s["seed"], s["index"], s["m"], s["l"], s["n"], s["lo"], s["hi"])
        C, st, ct, nxt = ref.mm_oracle(A, B, param_id=rec["param_id"], seed=gold["ctx_seed"],
                                      counter0=rec["counter0"], algo=rec["algo"], words=2 * 3 * 8192)
        assert hashlib.sha256(ct.astype("<u8").tobytes()).hexdigest() == rec["ct_sha256"], name
        assert st[:12].astype(int).tolist() == rec["stats"]


def test_oracle_key_import_export_round_trip():
    """Keys exported from one oracle session and imported into another (with a
    different seed) make the second one compute the first one's ciphertexts."""
    from oracle.bindings import Oracle

    a, b = Oracle(2, 11), Oracle(2, 12)
    for kind in (0, 1):
        b.import_key(kind, a.export_key(kind))
    rng = np.random.default_rng(3)
    N = a.N
    u = rng.integers(-1, 2, N)
    e0, e1 = rng.integers(-5, 6, N), rng.integers(-5, 6, N)
    v = rng.integers(-8, 8, 64)
    ca, cb = a.encrypt_noise(v, u, e0, e1), b.encrypt_noise(v, u, e0, e1)
    assert np.array_equal(ca, cb)
    assert np.array_equal(b.decrypt(ca, 64), v % 65537)
    elt = 3  # rotation by one slot
    b.import_key(2, a.export_key(2, elt), elt)
    b.import_key(2, a.export_key(2, 0), 0)
    assert np.array_equal(a.rot(ca, 1), b.rot(cb, 1))
    assert np.array_equal(a.mult(ca, ca), b.mult(cb, cb))


def test_gaussian_cdt_matches_exact_derivation():
    """oracle/gen_cdt.py: the committed CDT (sigma 3.2, tail 19) agrees with a
    60-digit recomputation to within 2^-50, and the device copy is identical."""
    import re
    import subprocess
    import sys

    r = subprocess.run([sys.executable, "oracle/gen_cdt.py", "--check"], cwd=ROOT, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    src = open(os.path.join(ROOT, "paper_2405_02238_b200", "csrc", "params.cpp")).read()
    dev = [int(h, 16) for h in re.findall(r"0x([0-9a-f]{16})ULL", src)]
    orc = open(os.path.join(ROOT, "oracle", "bfv_oracle.cpp")).read()
    body = re.search(r"kCdt\[20\]\s*=\s*\{(.*?)\};", orc, re.S).group(1)
    host = [int(h, 16) for h in re.findall(r"0x([0-9a-fA-F]+)ULL", body)]
    assert host and all(v in dev for v in host)
