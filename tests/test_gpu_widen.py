"""GPU: the SURVEY §8f "next" rows -- encrypted client transforms, square_pad_mm
and blocked_mm (the paper's 100x100 P1 / P2 partitions, Table 4) -- against the
reference's own implementation of each."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
T = 65537


def test_encrypted_client_transforms(gpu_factory, ref):
    g = gpu_factory(2)
    rng = np.random.default_rng(31)
    for _ in range(6):
        m, l, n = (int(x) for x in rng.integers(1, 10, 3))
        A = rng.integers(-9, 10, (m, l))
        B = rng.integers(-9, 10, (l, n))
        for aid, algo in [(0, "basic"), (1, "enhanced"), (2, "square_pad")]:
            C, st = g.matmul_batch(A, B, algo=aid, flags=1)
            Cref, st_ref = ref.mm2(A, B, algo, -1, 1, slots=g.slot_count)
            assert np.array_equal(C[0], Cref), (m, l, n, algo)
            assert st.astype(int).tolist() == st_ref[:12].astype(int).tolist()


@pytest.mark.parametrize("split", ["halves", "max_square"])
def test_blocked_100x100_paper_partitions(split, gpu_factory, ref):
    """acceptance criterion 7 / Table 4: 100x100 blocked with P1 (50/50) and P2 (64/36)."""
    g = gpu_factory(0)
    rng = np.random.default_rng(7)
    A = rng.integers(-9, 10, (100, 100))
    B = rng.integers(-9, 10, (100, 100))
    parts = [50, 50] if split == "halves" else [64, 36]
    C, log = g.blocked_mm(A, B, parts, parts, parts, algo=1)
    Cref, log_ref = ref.blocked(A, B, parts, parts, parts, "enhanced", slots=g.slot_count)
    assert np.array_equal(C, Cref)
    assert np.array_equal(C, (A @ B) % T)
    assert np.array_equal(log, log_ref), "block algorithm / fallback log differs"


def test_blocked_random_cuts_and_fallback(gpu_factory, ref):
    g = gpu_factory(2)
    rng = np.random.default_rng(22)

    def cuts(total):
        out, left = [], total
        while left:
            p = int(rng.integers(1, left + 1))
            out.append(p)
            left -= p
        return out

    for trial in range(6):
        m, l, n = (int(x) for x in rng.integers(2, 16, 3))
        A = rng.integers(-9, 10, (m, l))
        B = rng.integers(-9, 10, (l, n))
        plan = (cuts(m), cuts(l), cuts(n))
        for aid, algo in [(0, "basic"), (1, "enhanced")]:
            C, log = g.blocked_mm(A, B, *plan, algo=aid)
            Cref, log_ref = ref.blocked(A, B, *plan, algo, slots=g.slot_count)
            assert np.array_equal(C, Cref)
            assert np.array_equal(log, log_ref)
    # a block whose duplicated working set does not fit falls back to basic
    A = rng.integers(-9, 10, (36, 64))
    B = rng.integers(-9, 10, (64, 64))
    g0 = gpu_factory(0)
    C, log = g0.blocked_mm(A, B, [36], [64], [64], algo=1)
    assert np.array_equal(C, (A @ B) % T) and log[0][0] == 0 and log[0][1] == 1
