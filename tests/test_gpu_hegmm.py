"""GPU HEGMM end to end: the batched program executor against (a) the reference
algorithms over the reference SlotBackend{N/2, 65537} (decrypted values) and
(b) the reference algorithms over the CPU BFV oracle (final ciphertext words,
bit-exact).  Inputs are the reference campaign's seeded draws."""
import numpy as np
import pytest

from paper_2405_02238_b200.workload import CONFIGS, batch, splitmix_matrices

pytestmark = pytest.mark.gpu
T = 65537


@pytest.mark.parametrize("algo,aid", [("enhanced", 1), ("basic", 0)])
def test_cfg1_bit_exact_vs_oracle(algo, aid, gpu_factory, ref):
    m, l, n, lo, hi, pid, _, _ = CONFIGS["cfg1"]
    A, B = splitmix_matrices(20240101, 0, m, l, n, lo, hi)
    g = gpu_factory(pid)
    C, words = g.matmul_batch(A, B, algo=aid, counter0=0, export=True)
    Cref, st_ref = ref.mm(A, B, algo, slots=g.slot_count)
    assert np.array_equal(C[0], Cref)
    assert np.array_equal(C[0], (A @ B) % T)
    Co, st_o, ct_o, _ = ref.mm_oracle(A, B, param_id=pid, seed=1, counter0=0, algo=algo, words=g.ct_words)
    assert np.array_equal(Co, Cref)
    assert np.array_equal(words[0], ct_o), "final ciphertext differs from the op-by-op oracle"


def test_random_shapes_small_params(gpu_factory, ref):
    g = gpu_factory(2)
    rng = np.random.default_rng(3)
    for trial in range(12):
        m, l, n = (int(x) for x in rng.integers(1, 13, 3))
        A = rng.integers(-9, 10, (m, l)).astype(np.int64)
        B = rng.integers(-9, 10, (l, n)).astype(np.int64)
        for aid, algo in [(0, "basic"), (1, "enhanced")]:
            C, st = g.matmul_batch(A, B, algo=aid)
            Cref, st_ref = ref.mm(A, B, algo, slots=g.slot_count)
            assert np.array_equal(C[0], Cref), (m, l, n, algo)
            assert np.array_equal(st, st_ref[:12]), (m, l, n, algo)


def test_batch_instances_match_single(gpu_factory, ref):
    g = gpu_factory(2)
    A, B = batch(7, 0, 5, 6, 5, 4, -8, 7)
    C, _ = g.matmul_batch(A, B, algo=0)
    for i in range(5):
        assert np.array_equal(C[i], (A[i] @ B[i]) % T)
    C1, w1 = g.matmul_batch(A[2:3], B[2:3], algo=0, counter0=2 * 3, export=True)
    C5, w5 = g.matmul_batch(A, B, algo=0, counter0=0, export=True)
    assert np.array_equal(w1[0], w5[2]), "lockstep batching changed a ciphertext"


def test_acceptance_exactness_sweep(gpu_factory):
    """Acceptance criterion 1 (proj/tests/acceptance/acceptance_main.cpp:36-60):
    500 random shapes in [1,16]^3, entries in [-9, 9]; basic_mm, enhanced_mm and
    square_pad_mm on the B200 all equal the integer product (mod t = 65537,
    which is exact here: |C| <= 16 * 81 < t / 2)."""
    g = gpu_factory(0)
    rng = np.random.default_rng(20240101)
    failures = []
    for trial in range(500):
        m, l, n = (int(x) for x in rng.integers(1, 17, 3))
        A = rng.integers(-9, 10, (m, l)).astype(np.int64)
        B = rng.integers(-9, 10, (l, n)).astype(np.int64)
        want = (A @ B) % T
        for aid in (0, 1, 2):
            C, _ = g.matmul_batch(A, B, algo=aid, counter0=3 * trial)
            if not np.array_equal(C[0], want):
                failures.append((m, l, n, aid))
    assert not failures, failures[:5]
