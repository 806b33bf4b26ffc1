"""GPU: the boundary's key material, host-sampled randomness and session
semantics (include/hegmm_b200.h hgm_key_*, hgm_encrypt_noise, hgm_flush,
context lifetime, concurrent counters).

North_star: "given identical host-sampled keys and noise, ciphertexts must be
bit-exact".  Here the keys are produced on the HOST by the CPU oracle from a
seed the GPU never sees, uploaded into a KEYLESS cloud context, and every
encryption's (u, e0, e1) is sampled by numpy; the cloud context never holds
the secret key."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
T = 65537


def host_noise(rng, N):
    u = rng.integers(-1, 2, N).astype(np.int64)
    e0 = np.clip(np.round(rng.normal(0, 3.2, N)), -19, 19).astype(np.int64)
    e1 = np.clip(np.round(rng.normal(0, 3.2, N)), -19, 19).astype(np.int64)
    return u, e0, e1


@pytest.mark.parametrize("pid", [2, 0])
def test_device_keys_equal_oracle_keys(pid, gpu_factory, oracle_factory):
    """The GPU's own key generation (seeded) equals the oracle's, key by key."""
    g, o = gpu_factory(pid), oracle_factory(pid)
    for kind in (0, 1):
        assert np.array_equal(g.export_key(kind), o.export_key(kind)), f"key kind {kind}"
    for z in (None, 1, -5, 77):
        elt = 0 if z is None else g.galois_element(z)
        assert np.array_equal(g.export_key(2, elt), o.export_key(2, elt)), f"switching key {elt}"


@pytest.mark.parametrize("pid", [2, 0])
def test_host_keys_and_noise_bit_exact(pid):
    import paper_2405_02238_b200 as hb
    from oracle.bindings import Oracle

    client = Oracle(pid, 777)  # host side: holds sk; keys derived from a seed the GPU never sees
    cloud = hb.Context(pid, seed=5, device=0, flags=hb.CTX_KEYLESS)
    assert not cloud.has_key(hb.KEY_SECRET) and not cloud.has_key(hb.KEY_PUBLIC)
    cloud.upload_key(hb.KEY_PUBLIC, client.export_key(1))
    offsets = [1, 7, -3, 0]
    for z in offsets:
        if z:
            elt = cloud.galois_element(z)
            cloud.upload_key(hb.KEY_SWITCH, client.export_key(2, elt), elt=elt)
    cloud.upload_key(hb.KEY_SWITCH, client.export_key(2, 0), elt=0)  # relinearisation
    rng = np.random.default_rng(300 + pid)
    S = 200
    a, b = rng.integers(-8, 8, S), rng.integers(-8, 8, S)
    na, nb = host_noise(rng, cloud.N), host_noise(rng, cloud.N)
    ca, cb = cloud.encrypt_noise(a, *na), cloud.encrypt_noise(b, *nb)
    oa, ob = client.encrypt_noise(a, *na), client.encrypt_noise(b, *nb)
    assert np.array_equal(cloud.export(ca), oa)
    assert np.array_equal(cloud.export(cb), ob)
    full = np.zeros(cloud.slot_count, np.int64)
    full[:S] = a
    r = cloud.he_rot(ca, 7)
    assert np.array_equal(cloud.export(r), client.rot(oa, 7))
    assert np.array_equal(client.decrypt(cloud.export(r), S), np.roll(full, -7)[:S] % T)
    m = cloud.he_mult(ca, cb)
    assert np.array_equal(cloud.export(m), client.mult(oa, ob))
    assert np.array_equal(client.decrypt(cloud.export(m), S), (a * b) % T)
    masks = rng.integers(0, 2, (len(offsets), S)).astype(np.int64)
    p = cloud.apply_plan(ca, offsets, masks)
    acc = None
    for z, mk in zip(offsets, masks):
        term = client.cmult_x(client.rot_x(oa, z), mk)
        acc = term if acc is None else client.add_any(acc, term)
    assert np.array_equal(cloud.export(p), client.plain(acc))
    # the cloud cannot decrypt, nor rotate by an offset it holds no key for
    with pytest.raises(hb.HEError, match="secret key"):
        cloud.decrypt(ca)
    with pytest.raises(hb.HEError, match="Galois element"):
        cloud.export(cloud.he_rot(ca, 11))
    cloud.close()


def test_uploaded_keys_reproduce_golden_product(gpu_factory):
    """A keyless context given the oracle's seed-1 keys runs the cfg1 product
    to the ciphertext pinned in tests/golden/ciphertext_golden.json."""
    import hashlib
    import json
    import os

    import paper_2405_02238_b200 as hb
    from oracle.bindings import Oracle
    from paper_2405_02238_b200.workload import splitmix_matrices

    gold = {r["case"]: r for r in json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                                              "ciphertext_golden.json")))["cases"]}
    rec = gold["cfg1/enhanced"]
    o = Oracle(0, 1)
    g = hb.Context(0, seed=1, device=0, flags=hb.CTX_KEYLESS)
    for kind in (0, 1):
        g.upload_key(kind, o.export_key(kind))
    s = rec["inputs"]
    elts = hb.program_keys(1, s["m"], s["l"], s["n"], g.slot_count, g.N)
    for elt in elts:
        g.upload_key(hb.KEY_SWITCH, o.export_key(2, elt), elt=elt)
    A, B = splitmix_matrices(s["seed"], s["index"], s["m"], s["l"], s["n"], s["lo"], s["hi"])
    C, words = g.matmul_batch(A, B, algo=1, counter0=0, export=True)
    assert np.array_equal(C[0], (A @ B) % T)
    assert hashlib.sha256(words[0].astype("<u8").tobytes()).hexdigest() == rec["ct_sha256"]
    g.close()


def test_key_upload_validation(gpu_factory):
    import paper_2405_02238_b200 as hb

    g = hb.Context(2, seed=3, device=0, flags=hb.CTX_KEYLESS)
    pk = np.zeros(g.key_words(hb.KEY_PUBLIC), np.uint64)
    with pytest.raises(hb.HEError, match="size"):
        g.upload_key(hb.KEY_PUBLIC, pk[:-1])
    pk[5] = np.uint64(2**63)
    with pytest.raises(hb.HEError, match="canonical"):
        g.upload_key(hb.KEY_PUBLIC, pk)
    with pytest.raises(hb.HEError, match="Galois element"):
        g.upload_key(hb.KEY_SWITCH, np.zeros(g.key_words(2), np.uint64), elt=4)
    with pytest.raises(hb.HEError, match="public key"):
        g.encrypt([1, 2, 3])
    g.close()


def test_drop_secret_makes_a_cloud_context(gpu_factory):
    import paper_2405_02238_b200 as hb

    g = hb.Context(2, seed=8, device=0)
    ct = g.encrypt([3, 4, 5], counter=1)
    assert g.has_key(hb.KEY_SECRET)
    r = g.he_rot(ct, 1)
    g.export(r)  # key for offset 1 generated while sk was present
    g.drop_secret()
    assert not g.has_key(hb.KEY_SECRET)
    g.export(g.he_rot(ct, 1))  # existing key still usable
    with pytest.raises(hb.HEError, match="secret key"):
        g.decrypt(ct)
    with pytest.raises(hb.HEError, match="Galois element"):
        g.export(g.he_rot(ct, 2))
    g.close()


def test_concurrent_encrypt_never_reuses_randomness():
    """hgm_encrypt reserves its counter atomically: 4 threads x 16 encryptions
    of the same values on one context give 64 distinct c1 parts."""
    import paper_2405_02238_b200 as hb

    g = hb.Context(2, seed=9, device=0)
    out, lock = [], threading.Lock()

    def work():
        for _ in range(16):
            ct = g.encrypt([1, 2, 3])
            w = g.export(ct)
            with lock:
                out.append(w[g.ct_words // 2:].tobytes())

    ts = [threading.Thread(target=work) for _ in range(4)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    assert len(out) == 64 and len(set(out)) == 64
    # batch calls without an explicit counter0 also take fresh counters
    A = np.ones((1, 2, 2), np.int64)
    _, w1 = g.matmul_batch(A, A, algo=0, export=True)
    _, w2 = g.matmul_batch(A, A, algo=0, export=True)
    assert not np.array_equal(w1, w2)
    g.close()


def test_handles_outlive_closed_context():
    """Context.close() with live ciphertexts and batches: the native context
    stays alive until the last handle is released (no use-after-free)."""
    import gc

    import paper_2405_02238_b200 as hb

    g = hb.Context(2, seed=10, device=0)
    ct = g.encrypt([1, 2, 3], counter=0)
    r = g.he_rot(ct, 1)
    A = np.ones((2, 3, 3), np.int64)
    bt = hb.Batch(g, A, A, algo=0, counter0=0)
    g.close()
    del ct, r
    gc.collect()
    bt.free()
    g2 = hb.Context(2, seed=10, device=0)
    assert np.array_equal(g2.decrypt(g2.encrypt([1, 2, 3], counter=0)), [1, 2, 3])
    g2.close()


def test_flush_materialises_pinned_pending_values(gpu_factory, oracle_factory):
    import paper_2405_02238_b200 as hb

    g, o = hb.Context(2, seed=1, device=0), oracle_factory(2)
    a = np.arange(10)
    ca = g.encrypt(a, counter=50)
    r = g.he_rot(ca, 3)
    n0 = g.launch_count()
    g.flush()
    n1 = g.launch_count()
    assert n1 > n0, "flush launched nothing"
    w = g.export(r)
    assert g.launch_count() == n1, "export recomputed a flushed value"
    assert np.array_equal(w, o.rot(o.encrypt(a, 50), 3))
    g.close()


def test_os_seeded_sessions_sample_from_chacha():
    """HGM_CTX_OS_SEED: keys and noise come from ChaCha12 keyed by the OS CSPRNG.
    Two sessions get independent keys, neither equals the parity PRF's keys for
    any small seed, the seed is not exported, and products stay exact."""
    import numpy as np

    import paper_2405_02238_b200 as hb
    from paper_2405_02238_b200.workload import batch

    a = hb.Context(2, 0, 0, flags=hb.CTX_OS_SEED)
    b = hb.Context(2, 0, 0, flags=hb.CTX_OS_SEED)
    try:
        info = np.zeros(64, dtype=np.uint64)
        hb._check(hb.lib().hgm_ctx_info(a._h, hb._ptr(info), 64))
        assert int(info[7]) == 0  # the seed is never exported
        pa, pb = a.export_key(hb.KEY_PUBLIC), b.export_key(hb.KEY_PUBLIC)
        assert not np.array_equal(pa, pb)
        for seed in (0, 1):  # not the splitmix parity keys of the seeds a caller might guess
            ref = hb.Context(2, seed, 0)
            try:
                assert not np.array_equal(ref.export_key(hb.KEY_PUBLIC), pa)
            finally:
                ref.close()
        A, B = batch(3, 0, 4, 8, 16, 4, -8, 7)
        C, _ = a.matmul_batch(A, B, algo=1)
        assert np.array_equal(C, np.einsum("kij,kjl->kil", A, B) % 65537)
        v = np.arange(-20, 20)
        ct1, ct2 = a.encrypt(v), a.encrypt(v)
        assert not np.array_equal(a.export(ct1), a.export(ct2))  # fresh noise per encryption
        assert np.array_equal(a.decrypt(ct1), v % 65537)
    finally:
        a.close()
        b.close()
