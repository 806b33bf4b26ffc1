"""TEST INFRASTRUCTURE ONLY: ctypes bindings of the CPU checkers.

* ``Oracle``  -- oracle/liboracle.so, the CPU RNS-BFV restatement (bfv_oracle.h).
* ``RefLib``  -- oracle/_ref/libhegmm_ref.so, the reference's own hot-path
  sources (matrix/backend/lintrans/algorithms.cpp) compiled in place, with the
  C shim in oracle/ref_shim.cpp.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module, and only as the checker / the CPU baseline.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhegmm_ref.so")

_vp, _sz, _u64, _i64, _int = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int


def _p(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


class OracleError(RuntimeError):
    pass


class Oracle:
    _lib = None

    @classmethod
    def lib(cls):
        if cls._lib is None:
            L = ctypes.CDLL(ORACLE_SO)
            L.orc_create.restype = _vp
            L.orc_create.argtypes = [_int, _u64]
            L.orc_destroy.argtypes = [_vp]
            L.orc_info.argtypes = [_vp, _vp, _sz]
            L.orc_ct_words.restype = _sz
            L.orc_ct_words.argtypes = [_vp]
            L.orc_last_error.restype = ctypes.c_char_p
            L.orc_pending_words.restype = _sz
            L.orc_pending_words.argtypes = [_vp]
            L.orc_kind_words.restype = _sz
            L.orc_kind_words.argtypes = [_vp, _int]
            for name, args in {
                "orc_encrypt": [_vp, _vp, _sz, _u64, _vp],
                "orc_decrypt": [_vp, _vp, _sz, _vp],
                "orc_add": [_vp, _vp, _vp, _vp],
                "orc_cmult": [_vp, _vp, _vp, _sz, _vp],
                "orc_rot": [_vp, _vp, _i64, _vp],
                "orc_mult": [_vp, _vp, _vp, _vp],
                "orc_mult_pending": [_vp, _vp, _vp, _vp],
                "orc_add_any": [_vp, _vp, _int, _vp, _int, _vp],
                "orc_materialize": [_vp, _vp, _vp],
                "orc_materialize_kind": [_vp, _vp, _int, _vp],
                "orc_rot_x": [_vp, _vp, _i64, _vp, _vp],
                "orc_cmult_x": [_vp, _vp, _int, _vp, _sz, _vp, _vp],
                "orc_ntt_fwd": [_vp, _int, _vp],
                "orc_ntt_inv": [_vp, _int, _vp],
                "orc_encode": [_vp, _vp, _sz, _vp],
                "orc_key_export": [_vp, _int, ctypes.c_uint32, _vp],
                "orc_key_import": [_vp, _int, ctypes.c_uint32, _vp],
                "orc_encrypt_noise": [_vp, _vp, _sz, _vp, _vp, _vp, _vp],
            }.items():
                fn = getattr(L, name)
                fn.restype = _int
                fn.argtypes = args
            L.orc_key_words.restype = _sz
            L.orc_key_words.argtypes = [_vp, _int]
            L.orc_noise_budget.restype = ctypes.c_double
            L.orc_noise_budget.argtypes = [_vp, _vp]
            L.orc_prng.restype = _u64
            L.orc_prng.argtypes = [_u64, _u64, _u64]
            L.orc_gauss.restype = _i64
            L.orc_gauss.argtypes = [_u64, _u64, _u64]
            cls._lib = L
        return cls._lib

    def __init__(self, param_id: int = 0, seed: int = 1):
        L = self.lib()
        self._h = L.orc_create(param_id, seed)
        if not self._h:
            raise OracleError(L.orc_last_error().decode())
        info = np.zeros(64, dtype=np.uint64)
        L.orc_info(self._h, _p(info), 64)
        self.N, self.L, self.K, self.nB, self.dnum, self.t = (int(x) for x in info[:6])
        self.primes = [int(x) for x in info[8:8 + self.L + self.K + self.nB]]
        self.words = int(L.orc_ct_words(self._h))

    def __del__(self):
        try:
            if self._h:
                self.lib().orc_destroy(self._h)
        except Exception:
            pass

    def _chk(self, rc):
        if rc != 0:
            raise OracleError(self.lib().orc_last_error().decode())

    def _ct(self):
        return np.zeros(self.words, dtype=np.uint64)

    def export_key(self, kind: int, elt: int = 0) -> np.ndarray:
        w = np.zeros(self.lib().orc_key_words(self._h, kind), dtype=np.uint64)
        self._chk(self.lib().orc_key_export(self._h, kind, elt, _p(w)))
        return w

    def import_key(self, kind: int, words, elt: int = 0) -> None:
        w = np.ascontiguousarray(words, dtype=np.uint64)
        assert w.size == self.lib().orc_key_words(self._h, kind)
        self._chk(self.lib().orc_key_import(self._h, kind, elt, _p(w)))

    def encrypt_noise(self, values, u, e0, e1) -> np.ndarray:
        v = np.ascontiguousarray(values, dtype=np.int64)
        uu, a, b = (np.ascontiguousarray(x, dtype=np.int64) for x in (u, e0, e1))
        out = self._ct()
        self._chk(self.lib().orc_encrypt_noise(self._h, _p(v), v.size, _p(uu), _p(a), _p(b), _p(out)))
        return out

    def encrypt(self, values, counter: int) -> np.ndarray:
        v = np.ascontiguousarray(values, dtype=np.int64)
        out = self._ct()
        self._chk(self.lib().orc_encrypt(self._h, _p(v), v.size, counter, _p(out)))
        return out

    def decrypt(self, ct: np.ndarray, S: int) -> np.ndarray:
        out = np.zeros(S, dtype=np.int64)
        self._chk(self.lib().orc_decrypt(self._h, _p(np.ascontiguousarray(ct)), S, _p(out)))
        return out

    def add(self, a, b):
        out = self._ct()
        self._chk(self.lib().orc_add(self._h, _p(a), _p(b), _p(out)))
        return out

    def cmult(self, a, mask):
        m = np.ascontiguousarray(mask, dtype=np.int64)
        out = self._ct()
        self._chk(self.lib().orc_cmult(self._h, _p(a), _p(m), m.size, _p(out)))
        return out

    def rot(self, a, z: int):
        out = self._ct()
        self._chk(self.lib().orc_rot(self._h, _p(a), int(z), _p(out)))
        return out

    def mult(self, a, b):
        out = self._ct()
        self._chk(self.lib().orc_mult(self._h, _p(a), _p(b), _p(out)))
        return out

    # Values with parts (bfv_oracle.cpp XCt): (words, kind), kind bits 1 = pending
    # product, 2 = pending key switch (0: plain words).  he_mult / he_rot /
    # he_cmult / he_add in this form are mult_pending / rot_x / cmult_x / add_any;
    # plain() materialises.
    def _buf(self, kind):
        return np.zeros(int(self.lib().orc_kind_words(self._h, int(kind))), dtype=np.uint64)

    def mult_pending(self, a, b):
        out = self._buf(1)
        self._chk(self.lib().orc_mult_pending(self._h, _p(a), _p(b), _p(out)))
        return (out, 1)

    def add_any(self, x, y):
        (a, ka), (b, kb) = x, y
        k = int(ka) | int(kb)
        out = self._buf(k)
        self._chk(self.lib().orc_add_any(self._h, _p(np.ascontiguousarray(a)), int(ka),
                                         _p(np.ascontiguousarray(b)), int(kb), _p(out)))
        return (out, k)

    def rot_x(self, a, z: int):
        out, k = self._buf(2), ctypes.c_int(0)
        self._chk(self.lib().orc_rot_x(self._h, _p(np.ascontiguousarray(a)), int(z), _p(out), ctypes.byref(k)))
        return (out[: int(self.lib().orc_kind_words(self._h, k.value))].copy(), k.value)

    def cmult_x(self, x, mask):
        a, ka = x
        m = np.ascontiguousarray(mask, dtype=np.int64)
        out, k = self._buf(int(ka) & 2), ctypes.c_int(0)
        self._chk(self.lib().orc_cmult_x(self._h, _p(np.ascontiguousarray(a)), int(ka), _p(m), m.size, _p(out),
                                         ctypes.byref(k)))
        return (out[: int(self.lib().orc_kind_words(self._h, k.value))].copy(), k.value)

    def plain(self, x):
        w, k = x
        if not k:
            return w[: self.words]
        out = self._ct()
        self._chk(self.lib().orc_materialize_kind(self._h, _p(np.ascontiguousarray(w)), int(k), _p(out)))
        return out

    def noise_budget(self, ct) -> float:
        return float(self.lib().orc_noise_budget(self._h, _p(np.ascontiguousarray(ct))))

    def ntt(self, data: np.ndarray, prime: int, forward: bool = True) -> np.ndarray:
        d = np.ascontiguousarray(data, dtype=np.uint64).copy()
        for k in range(d.size // self.N):
            view = d[k * self.N:(k + 1) * self.N]
            fn = self.lib().orc_ntt_fwd if forward else self.lib().orc_ntt_inv
            self._chk(fn(self._h, prime, _p(view)))
        return d

    def encode(self, values) -> np.ndarray:
        v = np.ascontiguousarray(values, dtype=np.int64)
        out = np.zeros(self.N, dtype=np.uint64)
        self._chk(self.lib().orc_encode(self._h, _p(v), v.size, _p(out)))
        return out


ALGO = {"basic": 0, "enhanced": 1, "square_pad": 2}


class RefLib:
    """The reference's own algorithms (compiled from /root/reference sources)."""

    _lib = None

    @classmethod
    def available(cls) -> bool:
        return os.path.exists(REF_SO)

    @classmethod
    def lib(cls):
        if cls._lib is None:
            L = ctypes.CDLL(REF_SO)
            L.ref_last_error.restype = ctypes.c_char_p
            L.ref_mm.restype = _int
            L.ref_mm.argtypes = [_int, _int, _vp, _sz, _sz, _vp, _sz, _sz, _i64, _vp, _vp]
            L.ref_naive_mod.restype = _int
            L.ref_naive_mod.argtypes = [_vp, _sz, _sz, _vp, _sz, _i64, _vp]
            L.ref_trace.restype = ctypes.c_long
            L.ref_trace.argtypes = [_int, _int, _vp, _sz, _sz, _vp, _sz, _sz, _vp, _sz, _vp, _sz, _vp]
            L.ref_mm_oracle.restype = ctypes.c_long
            L.ref_mm_oracle.argtypes = [_int, _u64, _u64, _int, _int, _vp, _sz, _sz, _vp, _sz, _vp, _vp, _vp]
            L.ref_mm2.restype = _int
            L.ref_mm2.argtypes = [_int, _int, _int, _vp, _sz, _sz, _vp, _sz, _sz, _i64, _vp, _vp]
            L.ref_trace2.restype = ctypes.c_long
            L.ref_trace2.argtypes = [_int, _int, _int, _vp, _sz, _sz, _vp, _sz, _sz, _vp, _sz, _vp, _sz, _vp]
            L.ref_blocked.restype = _int
            L.ref_blocked.argtypes = [_int, _vp, _sz, _vp, _sz, _vp, _sz, _vp, _sz, _sz, _vp, _sz, _sz, _i64, _vp,
                                      _vp]
            L.ref_campaign.restype = _int
            L.ref_campaign.argtypes = [_sz, _sz, _sz, _u64, _int, _sz, _i64, _vp, _vp, _vp, _vp, _vp]
            L.ref_oracle_session_create.restype = _vp
            L.ref_oracle_session_create.argtypes = [_int, _u64]
            L.ref_oracle_session_destroy.argtypes = [_vp]
            L.ref_oracle_session_mm.restype = ctypes.c_long
            L.ref_oracle_session_mm.argtypes = [_vp, _u64, _int, _int, _vp, _sz, _sz, _vp, _sz, _vp]
            cls._lib = L
        return cls._lib

    @classmethod
    def _err(cls):
        return cls.lib().ref_last_error().decode()

    @classmethod
    def mm(cls, A, B, algo="basic", order=-1, slots=4096, modulus=65537):
        A = np.ascontiguousarray(A, dtype=np.int64)
        B = np.ascontiguousarray(B, dtype=np.int64)
        m, l = A.shape
        n = B.shape[1]
        C = np.zeros((m, n), dtype=np.int64)
        st = np.zeros(13, dtype=np.uint64)
        rc = cls.lib().ref_mm(ALGO[algo], order, _p(A), m, l, _p(B), n, slots, modulus, _p(C), _p(st))
        if rc != 0:
            raise OracleError(f"rc={rc}: {cls._err()}")
        return C, st

    @classmethod
    def campaign(cls, cases, lo, hi, seed, algos_mask=7, slots=4096, modulus=65537):
        """The reference's run_campaign over SlotBackend: (shapes[c,3], costs[c,k,2],
        exact[c,k], stats[c,k,12], resampled), k over the algorithms in mask bit order."""
        k = bin(algos_mask).count("1")
        shapes = np.zeros((cases, 3), dtype=np.uint64)
        costs = np.zeros((cases, k, 2), dtype=np.float64)
        exact = np.zeros((cases, k), dtype=np.uint8)
        stats = np.zeros((cases, k, 12), dtype=np.uint64)
        res = np.zeros(1, dtype=np.uint64)
        rc = cls.lib().ref_campaign(cases, lo, hi, seed, algos_mask, slots, modulus, _p(shapes), _p(costs),
                                    _p(exact), _p(stats), _p(res))
        if rc != 0:
            raise OracleError(f"rc={rc}: {cls._err()}")
        return shapes, costs, exact, stats, int(res[0])

    @classmethod
    def mm2(cls, A, B, algo="basic", order=-1, flags=0, slots=4096, modulus=65537):
        A = np.ascontiguousarray(A, dtype=np.int64)
        B = np.ascontiguousarray(B, dtype=np.int64)
        m, l = A.shape
        n = B.shape[1]
        C = np.zeros((m, n), dtype=np.int64)
        st = np.zeros(13, dtype=np.uint64)
        rc = cls.lib().ref_mm2(ALGO[algo], order, flags, _p(A), m, l, _p(B), n, slots, modulus, _p(C), _p(st))
        if rc != 0:
            raise OracleError(f"rc={rc}: {cls._err()}")
        return C, st

    @classmethod
    def trace2(cls, A, B, algo="basic", order=-1, flags=0, slots=4096):
        A = np.ascontiguousarray(A, dtype=np.int64)
        B = np.ascontiguousarray(B, dtype=np.int64)
        m, l = A.shape
        n = B.shape[1]
        dl = ctypes.c_size_t()
        cnt = cls.lib().ref_trace2(ALGO[algo], order, flags, _p(A), m, l, _p(B), n, slots, None, 0, None, 0,
                                   ctypes.byref(dl))
        if cnt < 0:
            raise OracleError(cls._err())
        hdr = np.zeros(3 * cnt, dtype=np.int64)
        data = np.zeros(max(1, dl.value), dtype=np.int64)
        cls.lib().ref_trace2(ALGO[algo], order, flags, _p(A), m, l, _p(B), n, slots, _p(hdr), hdr.size, _p(data),
                             data.size, ctypes.byref(dl))
        return hdr.reshape(-1, 3), data[:dl.value]

    @classmethod
    def blocked(cls, A, B, rows, mids, cols, algo="enhanced", slots=4096, modulus=65537):
        A = np.ascontiguousarray(A, dtype=np.int64)
        B = np.ascontiguousarray(B, dtype=np.int64)
        m, l = A.shape
        n = B.shape[1]
        r, md, c = (np.ascontiguousarray(x, dtype=np.uint64) for x in (rows, mids, cols))
        C = np.zeros((m, n), dtype=np.int64)
        log = np.zeros((r.size * md.size * c.size, 4), dtype=np.int32)
        rc = cls.lib().ref_blocked(ALGO[algo], _p(r), r.size, _p(md), md.size, _p(c), c.size, _p(A), m, l, _p(B),
                                   n, slots, modulus, _p(C), _p(log))
        if rc != 0:
            raise OracleError(f"rc={rc}: {cls._err()}")
        return C, log

    @classmethod
    def naive_mod(cls, A, B, q=65537):
        A = np.ascontiguousarray(A, dtype=np.int64)
        B = np.ascontiguousarray(B, dtype=np.int64)
        C = np.zeros((A.shape[0], B.shape[1]), dtype=np.int64)
        rc = cls.lib().ref_naive_mod(_p(A), A.shape[0], A.shape[1], _p(B), B.shape[1], q, _p(C))
        if rc != 0:
            raise OracleError(cls._err())
        return C

    @classmethod
    def trace(cls, A, B, algo="basic", order=-1, slots=4096):
        A = np.ascontiguousarray(A, dtype=np.int64)
        B = np.ascontiguousarray(B, dtype=np.int64)
        m, l = A.shape
        n = B.shape[1]
        dl = ctypes.c_size_t()
        cnt = cls.lib().ref_trace(ALGO[algo], order, _p(A), m, l, _p(B), n, slots, None, 0, None, 0,
                                  ctypes.byref(dl))
        if cnt < 0:
            raise OracleError(cls._err())
        hdr = np.zeros(3 * cnt, dtype=np.int64)
        data = np.zeros(max(1, dl.value), dtype=np.int64)
        cls.lib().ref_trace(ALGO[algo], order, _p(A), m, l, _p(B), n, slots, _p(hdr), hdr.size, _p(data),
                            data.size, ctypes.byref(dl))
        return hdr.reshape(-1, 3), data[:dl.value]

    @classmethod
    def mm_oracle(cls, A, B, param_id=0, seed=1, counter0=0, algo="basic", order=-1, words=None):
        A = np.ascontiguousarray(A, dtype=np.int64)
        B = np.ascontiguousarray(B, dtype=np.int64)
        m, l = A.shape
        n = B.shape[1]
        C = np.zeros((m, n), dtype=np.int64)
        st = np.zeros(13, dtype=np.uint64)
        ct = np.zeros(words, dtype=np.uint64) if words else None
        nxt = cls.lib().ref_mm_oracle(param_id, seed, counter0, ALGO[algo], order, _p(A), m, l, _p(B), n,
                                      _p(C), _p(ct) if ct is not None else None, _p(st))
        if nxt < 0:
            raise OracleError(f"rc={nxt}: {cls._err()}")
        return C, st, ct, nxt


class OracleSession:
    """Reference algorithms over a persistent CPU-BFV oracle context (one per thread).
    The ctypes calls release the GIL, so threads run truly in parallel."""

    def __init__(self, param_id: int = 0, seed: int = 1):
        self._h = RefLib.lib().ref_oracle_session_create(param_id, seed)
        if not self._h:
            raise OracleError(RefLib._err())

    def mm(self, A, B, algo="basic", order=-1, counter0=0):
        A = np.ascontiguousarray(A, dtype=np.int64)
        B = np.ascontiguousarray(B, dtype=np.int64)
        m, l = A.shape
        n = B.shape[1]
        C = np.zeros((m, n), dtype=np.int64)
        nxt = RefLib.lib().ref_oracle_session_mm(self._h, counter0, ALGO[algo], order, _p(A), m, l, _p(B), n, _p(C))
        if nxt < 0:
            raise OracleError(f"rc={nxt}: {RefLib._err()}")
        return C

    def close(self):
        if self._h:
            RefLib.lib().ref_oracle_session_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
