"""GPU parity: every primitive of libhegmm_b200.so against the CPU BFV oracle,
bit-exact on the ciphertext words (same seed => same keys and noise), and
decrypted values against plain modular arithmetic.  All calls go through the C ABI."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

T = 65537


def rand_vals(rng, S, lo=-8, hi=8):
    return rng.integers(lo, hi, S).astype(np.int64)


@pytest.mark.parametrize("pid", [2, 0, 1])
def test_ntt_matches_oracle(pid, gpu_factory, oracle_factory):
    g, o = gpu_factory(pid), oracle_factory(pid)
    rng = np.random.default_rng(pid)
    for prime in [0, g.L - 1, g.L, len(g.primes) - 1, -1]:
        q = T if prime < 0 else g.primes[prime]
        data = (rng.integers(0, 2**63, 2 * g.N, dtype=np.uint64) % np.uint64(q)).astype(np.uint64)
        f_gpu = g.test_ntt(data, prime, True)
        f_orc = o.ntt(data, prime, True)
        assert np.array_equal(f_gpu, f_orc), f"forward NTT prime {prime}"
        i_gpu = g.test_ntt(f_gpu, prime, False)
        assert np.array_equal(i_gpu, data), f"inverse NTT prime {prime}"


@pytest.mark.parametrize("pid", [0, 1])
def test_ntt_many_limbs(pid, gpu_factory, oracle_factory):
    """A launch of several waves (N = 32768: 4-CTA clusters, DSMEM outer stages):
    every limb's forward transform equals the oracle's, and inverse o forward
    is the identity on all of them."""
    g, o = gpu_factory(pid), oracle_factory(pid)
    rng = np.random.default_rng(77 + pid)
    count = 1500 if g.N == 8192 else 600
    prime = g.L - 1
    q = g.primes[prime]
    data = (rng.integers(0, 2**63, count * g.N, dtype=np.uint64) % np.uint64(q)).astype(np.uint64)
    f_gpu = g.test_ntt(data, prime, True)
    for k in (0, count // 2, count - 1):
        sl = slice(k * g.N, (k + 1) * g.N)
        assert np.array_equal(f_gpu[sl], o.ntt(data[sl], prime, True)), f"limb {k}"
    assert np.array_equal(g.test_ntt(f_gpu, prime, False), data)


@pytest.mark.parametrize("pid", [2, 0])
def test_encrypt_bit_exact(pid, gpu_factory, oracle_factory):
    g, o = gpu_factory(pid), oracle_factory(pid)
    rng = np.random.default_rng(10 + pid)
    for S, ctr in [(1, 0), (37, 5), (g.slot_count, 123456)]:
        v = rand_vals(rng, S)
        ct = g.encrypt(v, counter=ctr)
        assert np.array_equal(g.export(ct), o.encrypt(v, ctr))
        assert np.array_equal(g.decrypt(ct), v % T)


@pytest.mark.parametrize("pid", [2, 0])
def test_ops_bit_exact(pid, gpu_factory, oracle_factory):
    g, o = gpu_factory(pid), oracle_factory(pid)
    rng = np.random.default_rng(20 + pid)
    S = 300
    a, b = rand_vals(rng, S), rand_vals(rng, S)
    ca, cb = g.encrypt(a, counter=1000), g.encrypt(b, counter=1001)
    oa, ob = o.encrypt(a, 1000), o.encrypt(b, 1001)
    # add
    s = g.he_add(ca, cb)
    assert np.array_equal(g.export(s), o.add(oa, ob))
    assert np.array_equal(g.decrypt(s), (a + b) % T)
    # cmult
    mask = rng.integers(0, 2, S).astype(np.int64)
    cm = g.he_cmult(ca, mask)
    assert np.array_equal(g.export(cm), o.cmult(oa, mask))
    assert np.array_equal(g.decrypt(cm), (a * mask) % T)
    # rotations (left, right, identity, wrap)
    full = np.zeros(g.slot_count, np.int64)
    full[:S] = a
    for z in [1, 5, -3, 0, g.slot_count + 2]:
        r = g.he_rot(ca, z)
        assert np.array_equal(g.export(r), o.rot(oa, z)), f"rot {z}"
        assert np.array_equal(g.decrypt(r), np.roll(full, -z)[:S] % T)
    # mult
    m = g.he_mult(ca, cb)
    assert np.array_equal(g.export(m), o.mult(oa, ob))
    assert np.array_equal(g.decrypt(m), (a * b) % T)
    assert m.depth() == 1


def test_apply_plan_fused_equals_op_by_op(gpu_factory, oracle_factory):
    """hgm_apply_plan (hoisted, fused) == the oracle's rot/cmult/add sequence
    (pending key switches: the masked sum is moded down once)."""
    g, o = gpu_factory(2), oracle_factory(2)
    rng = np.random.default_rng(5)
    S = 256
    a = rand_vals(rng, S)
    ca, oa = g.encrypt(a, counter=77), o.encrypt(a, 77)
    offsets = [-7, 0, 3, 11]
    masks = rng.integers(0, 2, (len(offsets), S)).astype(np.int64)
    res = g.apply_plan(ca, offsets, masks)
    acc = None
    for z, m in zip(offsets, masks):
        term = o.cmult_x(o.rot_x(oa, z), m)
        acc = term if acc is None else o.add_any(acc, term)
    assert np.array_equal(g.export(res), o.plain(acc))


@pytest.mark.parametrize("pid", [2, 0])
def test_pending_products_bit_exact(pid, gpu_factory, oracle_factory):
    """he_mult is a pending product and he_add sums pending tensors (oracle
    XCt): sums of products, mixed with plain addends, materialised in one
    flush or read back between flushes, masked or rotated afterwards."""
    g, o = gpu_factory(pid), oracle_factory(pid)
    rng = np.random.default_rng(40 + pid)
    S = 257
    v = [rand_vals(rng, S) for _ in range(6)]
    gc = [g.encrypt(x, counter=2000 + i) for i, x in enumerate(v)]
    oc = [(o.encrypt(x, 2000 + i), False) for i, x in enumerate(v)]
    # one flush: acc = c5 + c0 c1 + c2 c3 + c4 c4
    gacc, oacc = gc[5], oc[5]
    for i, j in [(0, 1), (2, 3), (4, 4)]:
        gacc = g.he_add(gacc, g.he_mult(gc[i], gc[j]))
        oacc = o.add_any(oacc, o.mult_pending(oc[i][0], oc[j][0]))
    want = (v[5] + v[0] * v[1] + v[2] * v[3] + v[4] * v[4]) % T
    assert np.array_equal(g.export(gacc), o.plain(oacc))
    assert np.array_equal(g.decrypt(gacc), want)
    # the flushed sum is still pending: adding another product sums tensors
    p2 = g.he_mult(gc[0], gc[5])
    gsum = g.he_add(p2, gacc)
    osum = o.add_any(o.mult_pending(oc[0][0], oc[5][0]), oacc)
    assert np.array_equal(g.export(gsum), o.plain(osum))
    # a product read twice: by a sum and by a mask product
    mask = rng.integers(0, 2, S).astype(np.int64)
    p01 = g.he_mult(gc[0], gc[1])
    gmix = g.he_add(g.he_cmult(p01, mask), g.he_add(p01, gc[2]))
    op01 = o.mult_pending(oc[0][0], oc[1][0])
    omix = o.add_any((o.cmult(o.plain(op01), mask), False), o.add_any(op01, oc[2]))
    assert np.array_equal(g.export(gmix), o.plain(omix))
    assert np.array_equal(g.decrypt(gmix), (v[0] * v[1] * mask + v[0] * v[1] + v[2]) % T)
    # identity and real rotations of a pending sum read its materialised value
    for z in (0, 3):
        r = g.he_rot(gacc, z)
        assert np.array_equal(g.export(r), o.rot(o.plain(oacc), z))
    # product of a pending value (materialised operand)
    m2 = g.he_mult(gacc, gc[1])
    assert np.array_equal(g.export(m2), o.mult(o.plain(oacc), oc[1][0]))


@pytest.mark.parametrize("pid", [2, 0])
def test_pending_key_switches_bit_exact(pid, gpu_factory, oracle_factory):
    """he_rot is a pending key switch (oracle XCt part A): masked sums of
    rotations are moded down once; values mixing plain, key-switch and product
    parts; reads between flushes; rotations and products of such values."""
    g, o = gpu_factory(pid), oracle_factory(pid)
    rng = np.random.default_rng(60 + pid)
    S = 300
    a, b = rand_vals(rng, S), rand_vals(rng, S)
    ga, gb = g.encrypt(a, counter=3000), g.encrypt(b, counter=3001)
    oa, ob = o.encrypt(a, 3000), o.encrypt(b, 3001)
    m = [rng.integers(0, 2, S).astype(np.int64) for _ in range(4)]
    # eps = m0 rot(a, 1) + m1 rot(a, 7) + m2 rot(a, -2)   (an apply_plan-like masked sum)
    geps, oeps = None, None
    for z, mk in [(1, m[0]), (7, m[1]), (-2, m[2])]:
        gt = g.he_cmult(g.he_rot(ga, z), mk)
        ot = o.cmult_x(o.rot_x(oa, z), mk)
        geps = gt if geps is None else g.he_add(geps, gt)
        oeps = ot if oeps is None else o.add_any(oeps, ot)
    assert oeps[1] == 2
    assert np.array_equal(g.export(geps), o.plain(oeps))
    full = np.zeros(g.slot_count, np.int64)
    full[:S] = a
    want = sum(np.roll(full, -z)[:S] * mk for z, mk in [(1, m[0]), (7, m[1]), (-2, m[2])]) % T
    assert np.array_equal(g.decrypt(geps), want)
    # the flushed sum keeps its parts: mask it again, add a plain value and a product
    gmix = g.he_add(g.he_add(g.he_cmult(geps, m[3]), gb), g.he_mult(ga, gb))
    omix = o.add_any(o.add_any(o.cmult_x(oeps, m[3]), (ob, 0)), o.mult_pending(oa, ob))
    assert omix[1] == 3
    assert np.array_equal(g.export(gmix), o.plain(omix))
    # masking a value with a product part reads it materialised
    gmm = g.he_cmult(gmix, m[0])
    assert np.array_equal(g.export(gmm), o.plain(o.cmult_x(omix, m[0])))
    # rotating / multiplying a non-plain value reads it materialised
    r = g.he_rot(gmix, 3)
    assert np.array_equal(g.export(r), o.rot(o.plain(omix), 3))
    r0 = g.he_add(g.he_rot(geps, 0), ga)  # identity rotation: the plain value
    assert np.array_equal(g.export(r0), o.add(o.plain(oeps), oa))
    pm = g.he_mult(geps, gb)
    assert np.array_equal(g.export(pm), o.mult(o.plain(oeps), ob))
