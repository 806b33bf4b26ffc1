"""CPU: the library's HEGMM programs issue exactly the reference's op stream.

The program builder in paper_2405_02238_b200/csrc/hegmm_algos.cpp re-implements
basic_mm / enhanced_mm / apply_plan (proj/src/algorithms.cpp:198-367,
proj/src/lintrans.cpp:433-461).  These tests compare, op by op, its recorded
stream (kind, rotation offset, every cmult mask, per-phase counts) against
  * the committed golden digests made by running the reference (tests/golden), and
  * a live trace of the reference compiled from source (oracle/_ref), when built.
No GPU is touched: program construction is host code in libhegmm_b200.so."""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2405_02238_b200 as hb
from paper_2405_02238_b200.workload import CONFIGS, splitmix_matrices

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def digest(hdr, data):
    h = hashlib.sha256()
    off = 0
    for kind, arg, dlen in hdr.tolist():
        h.update(np.array([kind, arg], dtype=np.int64).tobytes())
        if kind == 4:
            h.update(np.ascontiguousarray(data[off:off + dlen], dtype=np.int64).tobytes())
        off += dlen
    return h.hexdigest()


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg5"])
@pytest.mark.parametrize("algo", ["basic", "enhanced"])
def test_config_streams_match_golden(name, algo):
    g = GOLD["configs"][name]
    rec = g["algos"][algo]
    N = 2 * g["slots"]
    if "error" in rec:
        with pytest.raises(hb.CapacityError):
            hb.program_info(hb.ALGOS[algo], g["m"], g["l"], g["n"], g["slots"], N)
        return
    st, facts = hb.program_info(hb.ALGOS[algo], g["m"], g["l"], g["n"], g["slots"], N)
    assert st.astype(int).tolist() == rec["stats"]
    hdr, data = hb.program_stream(hb.ALGOS[algo], g["m"], g["l"], g["n"], g["slots"], N)
    assert hdr.shape[0] == rec["ops"]
    assert digest(hdr, data) == rec["stream_sha256"]


def test_plan_kats():
    for p in GOLD["plans"]:
        if p["kind"] == "eps":
            off, w = hb.plan_info(0, p["k"], p["m"], p["l"], p["n"], 0, p["m"] * p["n"])
        else:
            off, w = hb.plan_info(1, p["k"], p["l"], p["m"], p["n"], 0, p["m"] * p["n"])
        assert off == p["offsets"] and w == p["weights"], p["source"]


def test_capacity_and_dimension_errors():
    with pytest.raises(hb.CapacityError):  # m*n = 20 > 16 (test_algorithms.cpp:96-104)
        hb.program_info(0, 5, 3, 4, slots=16, N=32)
    with pytest.raises(hb.CapacityError):  # (36,64,64) duplication needs 4608 slots (:294-304)
        hb.program_info(1, 36, 64, 64)
    st, _ = hb.program_info(0, 36, 64, 64)  # the plain pipeline still fits
    assert st[3] == 64  # l CC-mults in the cloud
    with pytest.raises(hb.DimensionError):
        hb.program_info(0, 0, 3, 4)


def test_pinned_strategies():
    # select_strategy examples (test_algorithms.cpp:114-149) via the CC-mult counts
    assert hb.program_info(1, 2, 5, 7)[0][3] == 2
    assert hb.program_info(1, 5, 4, 2)[0][3] == 2
    assert hb.program_info(1, 4, 4, 4)[0][3] == 4
    assert hb.program_info(0, 2, 5, 7)[0][3] == 5


def test_live_reference_traces_random_shapes(ref):
    rng = np.random.default_rng(11)
    for trial in range(60):
        m, l, n = (int(x) for x in rng.integers(1, 17, 3))
        A = rng.integers(-9, 10, (m, l))
        B = rng.integers(-9, 10, (l, n))
        for algo in ("basic", "enhanced"):
            for order in (-1, 0, 1):
                rh, rd = ref.trace(A, B, algo, order, slots=4096)
                mh, md = hb.program_stream(hb.ALGOS[algo], m, l, n, 4096, 8192, order)
                assert np.array_equal(rh[:, 0], mh[:, 0]), (m, l, n, algo, order)
                rot = rh[:, 0] == 5
                assert np.array_equal(rh[rot, 1], mh[rot, 1])
                assert digest(rh, rd) == digest(mh, md), (m, l, n, algo, order)
                _, st_ref = ref.mm(A, B, algo, order, slots=4096)
                st, _ = hb.program_info(hb.ALGOS[algo], m, l, n, 4096, 8192, order)
                assert st.astype(int).tolist() == st_ref[:12].astype(int).tolist()


def test_golden_products_with_reference(ref):
    """Reference outputs recorded in the golden file are reproducible here."""
    for name in ("cfg1", "cfg2", "cfg3"):
        g = GOLD["configs"][name]
        A, B = splitmix_matrices(GOLD["seed"], 0, g["m"], g["l"], g["n"], g["lo"], g["hi"])
        C, _ = ref.mm(A, B, "basic", slots=g["slots"])
        assert hashlib.sha256(C.astype(np.int64).tobytes()).hexdigest() == g["algos"]["basic"]["C_sha256"]
        assert np.array_equal(C, (A @ B) % 65537)


def test_encrypted_client_transforms_and_square_pad_streams(ref):
    """MultiplyOptions::encrypted_client_transforms (algorithms.cpp:219-227,
    :279-301) and square_pad_mm (:369-388): same op stream as the reference,
    including the client-phase rotations and masks."""
    rng = np.random.default_rng(21)
    for trial in range(25):
        m, l, n = (int(x) for x in rng.integers(1, 11, 3))
        A = rng.integers(-9, 10, (m, l))
        B = rng.integers(-9, 10, (l, n))
        for algo in ("basic", "enhanced", "square_pad"):
            for flags in (0, 1):
                order = (-1, 0, 1)[trial % 3]
                rh, rd = ref.trace2(A, B, algo, order, flags, slots=4096)
                mh, md = hb.program_stream(hb.ALGOS[algo], m, l, n, 4096, 8192, order, flags)
                assert digest(rh, rd) == digest(mh, md), (m, l, n, algo, flags, order)
                _, st_ref = ref.mm2(A, B, algo, order, flags, slots=4096)
                st, _ = hb.program_info(hb.ALGOS[algo], m, l, n, 4096, 8192, order, flags)
                assert st.astype(int).tolist() == st_ref[:12].astype(int).tolist()
                if flags:
                    assert st[4] > 0  # client-phase cmults (test_algorithms.cpp:84-94)


def test_schedule_defers_moddown_and_rescale():
    """The compiled 64^3 and cfg3 programs (CPU only): rotations after CSE, and
    one ModDown per masked sum of rotations / one scale-and-round +
    relinearisation per product sum (pending key switches and products)."""
    import paper_2405_02238_b200 as hb

    for algo in (0, 1):
        _, f = hb.program_info(algo, 64, 64, 64)
        assert (f["rotations"], f["cc_mults"], f["moddowns"], f["rescales"]) == (189, 64, 126, 1)
    _, f = hb.program_info(0, 32, 128, 16)
    assert (f["rotations"], f["cc_mults"], f["moddowns"], f["rescales"]) == (1725, 128, 255, 1)
