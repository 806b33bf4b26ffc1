"""GPU: every BASELINE.json config end to end on the B200, against the
reference's recorded outputs (tests/golden, made by running the reference),
plus ciphertext bit-exactness at N = 32768 (config 5 parameters)."""
import hashlib
import json
import os

import numpy as np
import pytest

from paper_2405_02238_b200.workload import CONFIGS, batch, splitmix_matrices

pytestmark = pytest.mark.gpu
T = 65537
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def sha(C):
    return hashlib.sha256(np.ascontiguousarray(C, dtype=np.int64).tobytes()).hexdigest()


@pytest.mark.parametrize("name,algo", [("cfg2", "basic"), ("cfg2", "enhanced"), ("cfg3", "basic"),
                                       ("cfg5", "enhanced"), ("cfg5", "basic")])
def test_config_matches_reference(name, algo, gpu_factory):
    import paper_2405_02238_b200 as hb

    g = GOLD["configs"][name]
    pid = CONFIGS[name][5]
    ctx = gpu_factory(pid)
    A, B = splitmix_matrices(GOLD["seed"], 0, g["m"], g["l"], g["n"], g["lo"], g["hi"])
    C, st = ctx.matmul_batch(A, B, algo=hb.ALGOS[algo])
    rec = g["algos"][algo]
    assert sha(C[0]) == rec["C_sha256"], f"{name} {algo} differs from the reference"
    assert st.astype(int).tolist() == rec["stats"]
    assert np.array_equal(C[0], (A @ B) % T)


def test_cfg3_enhanced_is_capacity_rejected(gpu_factory):
    import paper_2405_02238_b200 as hb

    g = GOLD["configs"]["cfg3"]
    A, B = splitmix_matrices(GOLD["seed"], 0, g["m"], g["l"], g["n"], g["lo"], g["hi"])
    with pytest.raises(hb.CapacityError):
        gpu_factory(0).matmul_batch(A, B, algo=1)


def test_cfg4_batch_slice(gpu_factory):
    """A slice of the 4096-instance batch, every instance checked."""
    ctx = gpu_factory(0)
    A, B = batch(20240404, 100, 48, 64, 64, 64, -8, 7)
    for algo in (0, 1):
        C, _ = ctx.matmul_batch(A, B, algo=algo, counter0=100 * 3)
        for i in range(48):
            assert np.array_equal(C[i], (A[i] @ B[i]) % T), (algo, i)


def test_n32768_ops_bit_exact(gpu_factory, oracle_factory):
    g, o = gpu_factory(1), oracle_factory(1)
    rng = np.random.default_rng(32)
    S = 1000
    a, b = rng.integers(-4, 4, S), rng.integers(-4, 4, S)
    ca, cb = g.encrypt(a, counter=9), g.encrypt(b, counter=10)
    oa, ob = o.encrypt(a, 9), o.encrypt(b, 10)
    assert np.array_equal(g.export(ca), oa)
    r = g.he_rot(ca, 129)
    assert np.array_equal(g.export(r), o.rot(oa, 129))
    m = g.he_mult(ca, cb)
    assert np.array_equal(g.export(m), o.mult(oa, ob))
    assert np.array_equal(g.decrypt(m), (a * b) % T)


def test_cfg5_row_block_sharding(gpu_factory):
    """Config 5 split into 8 independent 16x128x128 HEGMM-Enhanced products
    (the per-GPU unit of the 8-GPU decomposition), run as one batch here."""
    import paper_2405_02238_b200 as hb
    from paper_2405_02238_b200.dist import row_blocks, sharded_matmul

    g = GOLD["configs"]["cfg5"]
    A, B = splitmix_matrices(GOLD["seed"], 0, g["m"], g["l"], g["n"], g["lo"], g["hi"])
    ctx = gpu_factory(1)
    st, facts = hb.program_info(1, 16, 128, 128, ctx.slot_count, ctx.N)
    assert st[3] == 16 and facts["segment"] == 16384  # p = 16 CC-mults, fits N = 32768
    C = sharded_matmul(ctx, A, B, 8, algo=1)
    assert sha(C) == g["algos"]["enhanced"]["C_sha256"]
    assert [c for _, c in row_blocks(128, 8)] == [16] * 8


@pytest.mark.parametrize("name,algo", [("cfg2", "basic"), ("cfg2", "enhanced"), ("cfg3", "basic"),
                                       ("cfg5", "enhanced")])
def test_noise_budget_margin(name, algo, gpu_factory, oracle_factory):
    """The product ciphertexts keep a healthy invariant-noise budget (oracle's
    SEAL-convention measure on the exported words), so the parameter sets carry
    every config's multiplicative depth with room to spare."""
    import paper_2405_02238_b200 as hb

    m, l, n, lo, hi, pid, _, _ = CONFIGS[name]
    A, B = splitmix_matrices(GOLD["seed"], 0, m, l, n, lo, hi)
    C, words = gpu_factory(pid).matmul_batch(A, B, algo=hb.ALGOS[algo], export=True)
    assert np.array_equal(C[0], (A @ B) % 65537)
    budget = oracle_factory(pid).noise_budget(words[0])
    assert budget > 20, f"{name} {algo}: only {budget:.1f} bits of noise budget left"
