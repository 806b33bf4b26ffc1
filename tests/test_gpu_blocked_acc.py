"""blocked_mm with encrypted accumulation (hgm_blocked_mm_ex).

The reference decrypts every block product and adds in cleartext
(/root/reference/proj/src/algorithms.cpp:485-490); here the products of each
output block are summed as ciphertexts on the GPU and each sum is decrypted
once.  Pinned: products equal the reference's blocked_mm (and A.B mod t), the
per-block algorithm / fallback log equals the reference's, every summed
ciphertext equals the sum (mod q) of the CPU oracle's block-product
ciphertexts under the same counters, shards of output blocks reproduce the
single run word for word, and the sharded path through the library's
communicator decrypts on the root."""
import numpy as np
import pytest

import paper_2405_02238_b200 as hb

pytestmark = pytest.mark.gpu

T = 65537


@pytest.mark.parametrize("split", ["halves", "max_square"])
def test_paper_partitions_encrypted_accumulation(split, gpu_factory, ref):
    g = gpu_factory(0)
    rng = np.random.default_rng(7)
    A = rng.integers(-9, 10, (100, 100))
    B = rng.integers(-9, 10, (100, 100))
    parts = [50, 50] if split == "halves" else [64, 36]
    C, log, ndec = g.blocked_mm_acc(A, B, parts, parts, parts, algo=1)
    Cref, log_ref = ref.blocked(A, B, parts, parts, parts, "enhanced", slots=g.slot_count)
    assert np.array_equal(C, Cref)
    assert np.array_equal(C, (A @ B) % T)
    assert np.array_equal(log, log_ref)
    # the reference decrypts each of the 8 block products; one decrypt per output
    # block and slot layout here (P2's fallback blocks carry a second layout)
    assert ndec == 4 if split == "halves" else 4 <= ndec < 8


def block_counters(rows, mids, cols, algo, slots, N, counter0=0):
    """Encryption counter base of every block product, reference loop order."""
    out, ctr = {}, counter0
    for bi, mm in enumerate(rows):
        for bj, nn in enumerate(cols):
            for bk, ll in enumerate(mids):
                used = algo
                if algo == 1:
                    try:
                        hb.program_info(1, mm, ll, nn, slots, N)
                    except hb.CapacityError:
                        used = 0
                out[(bi, bj, bk)] = (ctr, used)
                ctr += hb.program_info(used, mm, ll, nn, slots, N)[1]["encryptions"]
    return out


@pytest.mark.parametrize("algo", [0, 1])
def test_summed_ciphertexts_match_oracle(algo, gpu_factory, oracle_factory, ref):
    g, o = gpu_factory(2), oracle_factory(2)
    rng = np.random.default_rng(31 + algo)
    rows, mids, cols = [5, 7], [4, 3, 6], [6, 2]
    A = rng.integers(-8, 8, (sum(rows), sum(mids)))
    B = rng.integers(-8, 8, (sum(mids), sum(cols)))
    C, log, ndec, words, meta = g.blocked_mm_acc(A, B, rows, mids, cols, algo=algo, counter0=0, export=True)
    assert np.array_equal(C, (A @ B) % T)
    ctrs = block_counters(rows, mids, cols, algo, g.slot_count, g.N)
    ro, mo, co = (np.concatenate([[0], np.cumsum(x)]) for x in (rows, mids, cols))
    names = {0: "basic", 1: "enhanced"}
    seen = 0
    def layout(used, bm, bl, bn):
        f = hb.program_info(used, bm, bl, bn, g.slot_count, g.N)[1]
        return used, f["layout_rows"], f["layout_cols"], f["order"]

    for k in range(meta.shape[0]):
        ob, used, bm, bl, bn, order, terms, seg = (int(x) for x in meta[k])
        bi, bj = divmod(ob, len(cols))
        want, members = None, 0
        for bk in range(len(mids)):
            base, u = ctrs[(bi, bj, bk)]
            if layout(u, bm, mids[bk], bn) != layout(used, bm, bl, bn):
                continue  # another slot layout: another sum
            members += 1
            Ab = A[ro[bi]:ro[bi + 1], mo[bk]:mo[bk + 1]]
            Bb = B[mo[bk]:mo[bk + 1], co[bj]:co[bj + 1]]
            _, _, ct, _ = ref.mm_oracle(Ab, Bb, param_id=2, seed=1, counter0=base, algo=names[u], words=o.words)
            want = ct if want is None else o.add(want, ct)
            seen += 1
        assert members == terms
        assert np.array_equal(words[k], want), f"summed ciphertext of output block {ob} differs from the oracle"
    assert seen == len(rows) * len(cols) * len(mids)
    assert ndec == meta.shape[0] <= len(rows) * len(cols) * len(mids)


def test_output_block_shards_reproduce_the_full_run(gpu_factory):
    g = gpu_factory(2)
    rng = np.random.default_rng(5)
    rows, mids, cols = [6, 4], [5, 5], [3, 7]
    A = rng.integers(-8, 8, (10, 10))
    B = rng.integers(-8, 8, (10, 10))
    C, _, _, words, meta = g.blocked_mm_acc(A, B, rows, mids, cols, algo=1, counter0=100, export=True)
    parts = [g.blocked_mm_acc(A, B, rows, mids, cols, algo=1, counter0=100, out_range=r, export=True)
             for r in [(0, 1), (1, 2), (3, 1)]]
    assert np.array_equal(sum(p[0] for p in parts) % T, C)
    assert np.array_equal(np.concatenate([p[3] for p in parts]), words)
    assert np.array_equal(np.concatenate([p[4] for p in parts]), meta)
    # export only: nothing is decrypted
    Cz, _, nd, w2, _ = g.blocked_mm_acc(A, B, rows, mids, cols, algo=1, counter0=100, export="only")
    assert nd == 0 and not Cz.any() and np.array_equal(w2, words)


def test_blocked_sharded_through_comm(gpu_factory, tmp_path):
    from paper_2405_02238_b200.dist import blocked_mm_sharded

    g = gpu_factory(0)
    rng = np.random.default_rng(9)
    A = rng.integers(-9, 10, (100, 100))
    B = rng.integers(-9, 10, (100, 100))
    comm = hb.Comm(g, 0, 1, id_file=str(tmp_path / "id"))
    try:
        C, ndec = blocked_mm_sharded(g, A, B, [50, 50], [50, 50], [50, 50], algo=1, comm=comm)
    finally:
        comm.close()
    assert np.array_equal(C, (A @ B) % T) and ndec == 4
    C1, nd1 = blocked_mm_sharded(g, A, B, [50, 50], [50, 50], [50, 50], algo=1)
    assert np.array_equal(C1, C) and nd1 == 4


def test_plain_blocked_mm_unchanged_and_flags_checked(gpu_factory):
    g = gpu_factory(2)
    A = np.arange(12).reshape(3, 4) % 7
    B = np.arange(8).reshape(4, 2) % 5
    C, log = g.blocked_mm(A, B, [3], [2, 2], [2], algo=0)
    assert np.array_equal(C, (A @ B) % T)
    A64, B64 = (np.ascontiguousarray(x, dtype=np.int64) for x in (A, B))
    r, md, c = (np.array(x, dtype=np.uint64) for x in ([3], [2, 2], [1, 1]))
    Cout = np.zeros((3, 2), dtype=np.int64)
    P = hb._ptr

    def call(flags, first, count):
        return hb.lib().hgm_blocked_mm_ex(g._h, 0, 3, 4, 2, P(r), 1, P(md), 2, P(c), 2, P(A64), P(B64), P(Cout),
                                          0, flags, first, count, None, None, None, 0, None, None)

    assert call(0, 0, 1) == hb.HGM_EARG  # an output block range needs encrypted accumulation
    assert call(2, 0, 1) == hb.HGM_EARG  # export-only needs encrypted accumulation
    assert call(8, 0, 1) == hb.HGM_EARG  # unknown flag
    assert call(1, 0, 1) == hb.HGM_OK and np.array_equal(Cout[:, :1], ((A @ B) % T)[:, :1])
    assert not Cout[:, 1:].any()  # the other output block is left untouched
    assert call(1, 0, 2) == hb.HGM_OK and np.array_equal(Cout, (A @ B) % T)
