"""GPU: the hegmm::Backend contract, restated from the reference's own backend
tests (proj/tests/test_backend.cpp) for the B200 BFV backend.

Values are compared mod t = 65537 (decrypt returns [0, t), as SlotBackend{N/2,
65537} does).  Rotation acts on the whole N/2-slot row, so the segment-cyclic
wrap test (test_backend.cpp:93-100) is restated on a full row; SURVEY.md 8(c)
lists it among the tests that do not transfer for S < N/2."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

T = 65537
ADD, MULT_CC, MULT_CP, ROT, ENC, DEC = range(6)  # hgm_stats op order (backend.hpp:50-57)


def total(st, op):
    return int(st[2 * op] + st[2 * op + 1])


@pytest.fixture
def be(gpu_factory):
    return gpu_factory(0)


def vec(*xs):
    return np.array(xs, dtype=np.int64)


def test_encrypt_decrypt_round_trip(be):  # test_backend.cpp:25-39
    rng = np.random.default_rng(5)
    for _ in range(20):
        n = int(rng.integers(1, 4097))
        v = rng.integers(-1000, 1001, n).astype(np.int64)
        ct = be.encrypt(v)
        assert ct.segment_length() == n and ct.depth() == 0
        assert np.array_equal(be.decrypt(ct), v % T)


def test_encrypt_rejects_empty_and_oversized(be):  # :41-46
    import paper_2405_02238_b200 as hb

    with pytest.raises(hb.DimensionError):
        be.encrypt(np.zeros(0, np.int64))
    with pytest.raises(hb.CapacityError):
        be.encrypt(np.ones(be.slot_count + 1, np.int64))
    be.encrypt(np.ones(be.slot_count, np.int64))


def test_add_is_slotwise(be):  # :48-56
    import paper_2405_02238_b200 as hb

    x, y = be.encrypt(vec(1, 2, 3)), be.encrypt(vec(4, 5, 6))
    assert np.array_equal(be.decrypt(be.he_add(x, y)), vec(5, 7, 9))
    assert np.array_equal(be.decrypt(be.he_add(x, be.encrypt(vec(0, 0, 0)))), vec(1, 2, 3))
    with pytest.raises(hb.DimensionError):
        be.he_add(x, be.encrypt(vec(1)))


def test_mult_is_slotwise_and_adds_depth(be):  # :58-69
    import paper_2405_02238_b200 as hb

    x, y = be.encrypt(vec(1, 2, 3)), be.encrypt(vec(4, 5, 6))
    prod = be.he_mult(x, y)
    assert np.array_equal(be.decrypt(prod), vec(4, 10, 18)) and prod.depth() == 1
    same = be.he_mult(x, be.encrypt(vec(1, 1, 1)))
    assert np.array_equal(be.decrypt(same), vec(1, 2, 3)) and same.depth() == 1
    with pytest.raises(hb.DimensionError):
        be.he_mult(x, be.encrypt(vec(1, 2)))


def test_depth_tracks_cc_chain_only(be):  # :71-83
    x, y = be.encrypt(vec(1, 2)), be.encrypt(vec(3, 4))
    for _ in range(3):
        x = be.he_mult(x, y)
    assert x.depth() == 3
    assert np.array_equal(be.decrypt(x), vec(27, 128))
    masked = be.he_cmult(x, vec(1, 0))
    assert masked.depth() == 3
    summed = be.he_add(masked, be.he_cmult(y, vec(1, 1)))
    assert summed.depth() == 3
    assert np.array_equal(be.decrypt(summed), vec(30, 4))


def test_cmult_masks_slots(be):  # :85-91
    import paper_2405_02238_b200 as hb

    x = be.encrypt(vec(1, 2, 3))
    assert np.array_equal(be.decrypt(be.he_cmult(x, vec(0, 1, 0))), vec(0, 2, 0))
    assert np.array_equal(be.decrypt(be.he_cmult(x, vec(1, 1, 1))), vec(1, 2, 3))
    with pytest.raises(hb.DimensionError):
        be.he_cmult(x, vec(1, 1))


def test_rot_is_cyclic_over_the_row(be):  # :93-100 on a full row
    S = be.slot_count
    v = (np.arange(S, dtype=np.int64) * 7 + 10) % T
    x = be.encrypt(v)
    for z in (1, 0, -1, S, 5, -S + 3):
        assert np.array_equal(be.decrypt(be.he_rot(x, z)), np.roll(v, -z)), z


def test_rot_composes_additively(be):  # :102-115 on a full row
    rng = np.random.default_rng(9)
    v = rng.integers(0, 100, be.slot_count).astype(np.int64)
    ct = be.encrypt(v)
    for _ in range(6):
        a, b = (int(z) for z in rng.integers(-20, 20, 2))
        assert np.array_equal(be.decrypt(be.he_rot(be.he_rot(ct, a), b)), be.decrypt(be.he_rot(ct, a + b)))


def test_every_primitive_bumps_exactly_one_counter(be):  # :117-141
    x, y = be.encrypt(vec(1, 2)), be.encrypt(vec(3, 4))
    be.reset_stats()
    be.he_add(x, y)
    s = be.stats()
    assert total(s, ADD) == 1 and total(s, MULT_CC) + total(s, MULT_CP) + total(s, ROT) == 0
    be.he_mult(x, y)
    s = be.stats()
    assert total(s, MULT_CC) == 1 and total(s, MULT_CP) == 0
    be.he_cmult(x, vec(1, 0))
    s = be.stats()
    assert total(s, MULT_CP) == 1 and total(s, MULT_CC) == 1
    be.he_rot(x, 1)
    assert total(be.stats(), ROT) == 1


def test_phase_splits_counters(be):  # :143-160
    be.reset_stats()
    be.set_phase(0)
    x = be.encrypt(vec(1, 2))
    be.set_phase(1)
    be.he_add(be.he_rot(x, 1), x)
    be.set_phase(0)
    s = be.stats()
    assert s[2 * ENC] == 1 and s[2 * ROT + 1] == 1 and s[2 * ROT] == 0 and s[2 * ADD + 1] == 1


def test_reset_clears_counters(be):  # :162-168
    x = be.encrypt(vec(1))
    be.he_add(be.he_rot(x, 1), x)
    be.reset_stats()
    s = be.stats()
    assert total(s, ROT) + total(s, ADD) + total(s, ENC) == 0


def test_concurrent_counting_is_consistent(be):  # :193-212 (4 threads on one backend)
    x = be.encrypt(np.ones(be.slot_count, np.int64))  # full row: invariant under row rotation
    be.reset_stats()
    outs, errs = [], []

    def work():
        try:
            for _ in range(50):
                outs.append(be.he_rot(x, 1))
        except Exception as e:  # pragma: no cover - reported below
            errs.append(e)

    ts = [threading.Thread(target=work) for _ in range(4)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    assert not errs, errs
    assert total(be.stats(), ROT) == 200
    for ct in outs[:: 40]:
        assert np.array_equal(be.decrypt(ct), np.ones(be.slot_count, np.int64))


def test_peak_live_tracks_high_water(be):  # :214-226
    be.reset_stats()
    a, b = be.encrypt(vec(1)), be.encrypt(vec(2))
    c = be.he_add(a, b)
    assert be.peak_live_ciphertexts() >= 3
    del a, b, c
    peak = be.peak_live_ciphertexts()
    be.encrypt(vec(1))
    assert be.peak_live_ciphertexts() == peak


def test_wire_format_round_trip_and_validation(be, gpu_factory):
    """hgm_ct_serialize / hgm_ct_deserialize: bit-identical round trip that keeps
    segment, depth and phase; corrupted, truncated or foreign ciphertexts are
    rejected."""
    import paper_2405_02238_b200 as hb

    x, y = be.encrypt(vec(1, 2, 3)), be.encrypt(vec(4, 5, 6))
    prod = be.he_mult(x, y)
    data = be.serialize(prod)
    assert len(data) == 48 + 8 * be.ct_words and data[:4] == b"HGMC"
    back = be.deserialize(data)
    assert back.segment_length() == 3 and back.depth() == 1
    assert np.array_equal(be.export(back), be.export(prod))
    assert np.array_equal(be.decrypt(be.he_add(back, x)), vec(5, 12, 21))
    bad = bytearray(data)
    bad[100] ^= 1
    with pytest.raises(hb.HEError):
        be.deserialize(bytes(bad))
    with pytest.raises(hb.HEError):
        be.deserialize(data[:-8])
    other = gpu_factory(0, seed=2)  # another key set
    with pytest.raises(hb.HEError):
        other.deserialize(data)


def test_concurrent_flushes_on_one_backend(be):
    """Several threads encrypting, rotating, multiplying and decrypting on one
    backend at once: device work is serialised inside the library and every
    thread gets its own correct result."""
    S = be.slot_count
    errs = []

    def work(k):
        try:
            rng = np.random.default_rng(100 + k)
            for _ in range(4):
                v = rng.integers(0, 50, S).astype(np.int64)
                w = rng.integers(0, 50, S).astype(np.int64)
                x, y = be.encrypt(v), be.encrypt(w)
                r = be.he_mult(be.he_rot(x, k + 1), y)
                got = be.decrypt(r)
                if not np.array_equal(got, (np.roll(v, -(k + 1)) * w) % T):
                    errs.append(k)
        except Exception as e:  # pragma: no cover - reported below
            errs.append(repr(e))

    ts = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    assert not errs, errs
