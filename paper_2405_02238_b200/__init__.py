"""paper_2405_02238_b200 -- B200-native HE primitives behind the HEGMM backend contract.

Thin ctypes mirror of the C ABI in ``include/hegmm_b200.h`` (which itself
mirrors ``hegmm::Backend``, /root/reference/proj/include/hegmm/backend.hpp:107-127).
All arithmetic runs in ``libhegmm_b200.so`` (hand-written sm_100a CUDA); this
module only marshals host buffers.  There is no CPU fallback: importing the
module without the built library, or creating a context without a GPU, raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HGM_LIB") or os.path.join(_HERE, "libhegmm_b200.so")


def _nccl_wheel() -> Optional[str]:
    """The nvidia-nccl wheel's libnccl.so.2 when installed (the build torch also
    loads): the library binds NCCL lazily and prefers one copy per process."""
    import importlib.util

    try:
        spec = importlib.util.find_spec("nvidia.nccl")
    except (ImportError, ValueError):
        return None
    for base in (spec.submodule_search_locations or []) if spec else []:
        cand = os.path.join(base, "lib", "libnccl.so.2")
        if os.path.exists(cand):
            return cand
    return None


if not os.environ.get("HGM_NCCL_LIB"):
    _w = _nccl_wheel()
    if _w:
        os.environ["HGM_NCCL_LIB"] = _w

HGM_OK, HGM_EDIM, HGM_ECAP, HGM_EINTERNAL, HGM_EOVERFLOW, HGM_ECUDA, HGM_EARG = range(7)
PHASE_CLIENT, PHASE_CLOUD = 0, 1
# C ABI symbols declared in include/hegmm_b200.h
EXPORTS = (
    "hgm_ctx_create", "hgm_ctx_destroy", "hgm_last_error", "hgm_ctx_info", "hgm_slot_count",
    "hgm_ct_words", "hgm_encrypt", "hgm_encrypt_at", "hgm_decrypt", "hgm_add", "hgm_mul",
    "hgm_cmul", "hgm_rot", "hgm_apply_plan", "hgm_flush", "hgm_ct_export", "hgm_ct_import",
    "hgm_ct_wire_size", "hgm_ct_serialize", "hgm_ct_deserialize",
    "hgm_ct_segment", "hgm_ct_depth", "hgm_ct_phase", "hgm_ct_retain", "hgm_ct_release", "hgm_ct_set_pinned",
    "hgm_stats", "hgm_reset_stats", "hgm_peak_live", "hgm_set_phase", "hgm_phase",
    "hgm_matmul_batch", "hgm_matmul_batch_export", "hgm_bench_ntt", "hgm_device_sync",
    "hgm_test_ntt", "hgm_launch_count", "hgm_batch_encrypt", "hgm_batch_cloud", "hgm_batch_output",
    "hgm_batch_decrypt", "hgm_batch_decrypt_words", "hgm_batch_free", "hgm_program_info",
    "hgm_program_stream", "hgm_plan_info", "hgm_blocked_mm",
    "hgm_ctx_create_ex", "hgm_key_words", "hgm_key_export", "hgm_key_upload", "hgm_key_drop_secret",
    "hgm_key_has", "hgm_galois_element", "hgm_encrypt_noise", "hgm_reserve_counters", "hgm_program_keys",
    "hgm_decrypt_products", "hgm_comm_unique_id", "hgm_comm_init", "hgm_comm_init_file", "hgm_comm_destroy",
    "hgm_comm_rank", "hgm_comm_size", "hgm_comm_barrier", "hgm_comm_max", "hgm_comm_gather",
    "hgm_comm_gather_batch", "hgm_comm_buffer_free", "hgm_bench_keyswitch", "hgm_blocked_mm_ex",
    "hgm_test_chacha", "hgm_bench_keyswitch_plan",
)
CTX_KEYLESS, CTX_OS_SEED = 1, 2
COUNTER_AUTO = (1 << 64) - 1
KEY_SECRET, KEY_PUBLIC, KEY_SWITCH = 0, 1, 2
FLAG_ENCRYPTED_CLIENT_TRANSFORMS = 1
ALGOS = {"basic": 0, "enhanced": 1, "square_pad": 2}


def plan_info(kind: int, k: int, a: int, b: int, c: int, order: int, segment: int):
    """(offsets, weights) of a diagonal plan (CPU only); see hgm_plan_info."""
    off = np.zeros(4096, dtype=np.int64)
    w = np.zeros(4096, dtype=np.uint64)
    cnt = lib().hgm_plan_info(kind, k, a, b, c, order, segment, _ptr(off), _ptr(w), off.size)
    if cnt < 0:
        _check(-cnt)
    return off[:cnt].tolist(), w[:cnt].astype(int).tolist()


def chacha_block(key, nonce: int, counter: int, rounds: int = 20) -> np.ndarray:
    """The ChaCha block function OS-seeded sessions sample from (test hook, CPU)."""
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(16, dtype=np.uint32)
    _check(lib().hgm_test_chacha(_ptr(k), nonce, counter, rounds, _ptr(out)))
    return out


def program_info(algo: int, m: int, l: int, n: int, slots: int = 4096, N: int = 8192, order: int = -1,
                 flags: int = 0):
    """Op counts (stats[12]) and facts of a compiled HEGMM program (CPU only)."""
    st = np.zeros(12, dtype=np.uint64)
    facts = np.zeros(11, dtype=np.uint64)
    _check(lib().hgm_program_info(algo, order, flags, m, l, n, slots, N, _ptr(st), _ptr(facts)))
    keys = ("segment", "encryptions", "rotations", "masked_sums", "cc_mults", "levels", "order", "moddowns",
            "rescales", "layout_rows", "layout_cols")
    return st, dict(zip(keys, (int(x) for x in facts)))


def program_keys(algo: int, m: int, l: int, n: int, slots: int = 4096, N: int = 8192, order: int = -1,
                 flags: int = 0):
    """Switching keys a product shape needs: Galois elements, 0 = relinearisation."""
    out = np.zeros(8192, dtype=np.uint32)
    cnt = lib().hgm_program_keys(algo, order, flags, m, l, n, slots, N, _ptr(out), out.size)
    if cnt < 0:
        _check(-cnt)
    return [int(x) for x in out[:cnt]]


def program_stream(algo: int, m: int, l: int, n: int, slots: int = 4096, N: int = 8192, order: int = -1,
                   flags: int = 0):
    """The recorded op stream (reference trace layout): (hdr[k,3], mask data)."""
    dl = ctypes.c_size_t()
    cnt = lib().hgm_program_stream(algo, order, flags, m, l, n, slots, N, None, 0, None, 0, ctypes.byref(dl))
    if cnt < 0:
        _check(-cnt)
    hdr = np.zeros(3 * cnt, dtype=np.int64)
    data = np.zeros(max(1, dl.value), dtype=np.int64)
    cnt2 = lib().hgm_program_stream(algo, order, flags, m, l, n, slots, N, _ptr(hdr), hdr.size, _ptr(data),
                                    data.size, ctypes.byref(dl))
    if cnt2 < 0:
        _check(-cnt2)
    return hdr.reshape(-1, 3), data[:dl.value]


class Batch:
    """Encrypted inputs of `count` instances resident in HBM (client phase done)."""

    def __init__(self, ctx: "Context", A: np.ndarray, B: np.ndarray, algo: int = 0, order: int = -1,
                 counter0: Optional[int] = None, flags: int = 0):
        A = _as_i64(A)
        B = _as_i64(B)
        if A.ndim == 2:
            A, B = A[None], B[None]
        self.ctx = ctx
        self.count, self.m, self.l = A.shape
        self.n = B.shape[2]
        h = ctypes.c_void_p()
        _check(lib().hgm_batch_encrypt(ctx._h, algo, order, flags, self.m, self.l, self.n, self.count,
                                       _ptr(A), _ptr(B), _counter(counter0), ctypes.byref(h)))
        self._h = h.value

    def cloud(self) -> float:
        """Run the cloud phase; returns its CUDA-event time in ms."""
        ms = ctypes.c_float()
        _check(lib().hgm_batch_cloud(self.ctx._h, self._h, ctypes.byref(ms)))
        return ms.value

    def output_ptr(self, i: int) -> int:
        return lib().hgm_batch_output(self._h, i)

    def decrypt(self) -> np.ndarray:
        C = np.zeros((self.count, self.m, self.n), dtype=np.int64)
        _check(lib().hgm_batch_decrypt(self.ctx._h, self._h, _ptr(C)))
        return C

    def free(self) -> None:
        if self._h:
            lib().hgm_batch_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Comm:
    """The session's NCCL communicator (include/hegmm_b200.h, hgm_comm_*): one
    process per GPU; moves result ciphertexts and control values only."""

    def __init__(self, ctx: "Context", rank: int, world: int, id_file: Optional[str] = None,
                 unique_id: Optional[bytes] = None, timeout_s: float = 120.0):
        self.ctx = ctx
        h = ctypes.c_void_p()
        if unique_id is not None:
            buf = ctypes.create_string_buffer(bytes(unique_id), 128)
            _check(lib().hgm_comm_init(ctx._h, rank, world, buf, ctypes.byref(h)))
        else:
            if id_file is None:
                raise ValueError("Comm needs id_file or unique_id")
            _check(lib().hgm_comm_init_file(ctx._h, rank, world, id_file.encode(), timeout_s, ctypes.byref(h)))
        self._h = h.value
        self.rank, self.world = rank, world

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(lib().hgm_comm_unique_id(buf))
        return buf.raw

    def barrier(self) -> None:
        _check(lib().hgm_comm_barrier(self._h))

    def max(self, x: float) -> float:
        v = ctypes.c_double(float(x))
        _check(lib().hgm_comm_max(self._h, ctypes.byref(v)))
        return v.value

    def gather_batch(self, batch: Optional["Batch"], root: int = 0):
        """Every rank's batch results to `root` (rank order): (device pointer,
        count) on the root -- free with free_buffer -- and (None, 0) elsewhere."""
        p = ctypes.c_void_p()
        n = ctypes.c_size_t()
        _check(lib().hgm_comm_gather_batch(self._h, batch._h if batch is not None else None, root,
                                           ctypes.byref(p), ctypes.byref(n)))
        return (p.value, n.value) if p.value else (None, 0)

    def gather_words(self, words: np.ndarray, total_cap: int = 0, root: int = 0) -> Optional[np.ndarray]:
        """Host uint64 words of every rank to `root` in rank order (staged through
        device memory by the library); total_cap = receive capacity on the root."""
        w = np.ascontiguousarray(words, dtype=np.uint64).ravel()
        recv = np.zeros(max(1, total_cap), dtype=np.uint64) if self.rank == root else None
        got = ctypes.c_size_t()
        _check(lib().hgm_comm_gather(self._h, _ptr(w) if w.size else None, w.size,
                                     _ptr(recv) if recv is not None else None, total_cap if recv is not None else 0,
                                     root, ctypes.byref(got)))
        return recv[: got.value] if self.rank == root else None

    def free_buffer(self, ptr: Optional[int]) -> None:
        if ptr:
            _check(lib().hgm_comm_buffer_free(self._h, ptr))

    def close(self) -> None:
        if self._h:
            lib().hgm_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HEError(RuntimeError):
    """Base error (reference hegmm::Error, errors.hpp:10-14)."""


class DimensionError(HEError):
    """Operand shapes are incompatible (errors.hpp:17-21)."""


class CapacityError(HEError):
    """Working set exceeds the slot budget (errors.hpp:23-27)."""


class OverflowError_(HEError):
    """Exact arithmetic would overflow (errors.hpp:29-33)."""


_ERRORS = {HGM_EDIM: DimensionError, HGM_ECAP: CapacityError, HGM_EOVERFLOW: OverflowError_}

_lib: Optional[ctypes.CDLL] = None
_vp, _sz, _u64, _i64, _int = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int


def lib() -> ctypes.CDLL:
    """Load the CUDA library (raises if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing; run `make -C paper_2405_02238_b200` "
                          "(or __graft_entry__.build()) first -- there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    sig = {
        "hgm_ctx_create": (_vp, [_int, _u64, _int]),
        "hgm_ctx_destroy": (None, [_vp]),
        "hgm_last_error": (ctypes.c_char_p, []),
        "hgm_ctx_info": (_int, [_vp, _vp, _sz]),
        "hgm_slot_count": (_sz, [_vp]),
        "hgm_ct_words": (_sz, [_vp]),
        "hgm_encrypt": (_int, [_vp, _vp, _sz, _vp]),
        "hgm_encrypt_at": (_int, [_vp, _vp, _sz, _u64, _vp]),
        "hgm_decrypt": (_int, [_vp, _vp, _vp, _sz]),
        "hgm_add": (_int, [_vp, _vp, _vp, _vp]),
        "hgm_mul": (_int, [_vp, _vp, _vp, _vp]),
        "hgm_cmul": (_int, [_vp, _vp, _vp, _sz, _vp]),
        "hgm_rot": (_int, [_vp, _vp, _i64, _vp]),
        "hgm_apply_plan": (_int, [_vp, _vp, _sz, _vp, _vp, _sz, _vp]),
        "hgm_flush": (_int, [_vp]),
        "hgm_ct_export": (_int, [_vp, _vp, _vp]),
        "hgm_ct_import": (_int, [_vp, _vp, _sz, _sz, _vp]),
        "hgm_ct_wire_size": (_sz, [_vp]),
        "hgm_ct_serialize": (_int, [_vp, _vp, _vp, _sz]),
        "hgm_ct_deserialize": (_int, [_vp, _vp, _sz, _vp]),
        "hgm_ct_segment": (_sz, [_vp]),
        "hgm_ct_depth": (_sz, [_vp]),
        "hgm_ct_phase": (_int, [_vp]),
        "hgm_ct_retain": (_vp, [_vp]),
        "hgm_ct_release": (None, [_vp]),
        "hgm_ct_set_pinned": (_int, [_vp, _int]),
        "hgm_stats": (_int, [_vp, _vp]),
        "hgm_reset_stats": (_int, [_vp]),
        "hgm_peak_live": (_sz, [_vp]),
        "hgm_set_phase": (_int, [_vp, _int]),
        "hgm_phase": (_int, [_vp]),
        "hgm_matmul_batch": (_int, [_vp, _int, _int, _int, _sz, _sz, _sz, _sz, _vp, _vp, _vp, _u64, _vp]),
        "hgm_matmul_batch_export": (_int, [_vp, _int, _int, _int, _sz, _sz, _sz, _sz, _vp, _vp, _vp, _u64, _vp]),
        "hgm_blocked_mm": (_int, [_vp, _int, _sz, _sz, _sz, _vp, _sz, _vp, _sz, _vp, _sz, _vp, _vp, _vp, _u64, _vp]),
        "hgm_blocked_mm_ex": (_int, [_vp, _int, _sz, _sz, _sz, _vp, _sz, _vp, _sz, _vp, _sz, _vp, _vp, _vp, _u64,
                                     _int, _sz, _sz, _vp, _vp, _vp, _sz, _vp, _vp]),
        "hgm_bench_ntt": (_int, [_vp, _int, _sz, _int, _vp]),
        "hgm_device_sync": (_int, [_vp]),
        "hgm_bench_keyswitch": (_int, [_vp, _sz, _int, _vp]),
        "hgm_bench_keyswitch_plan": (_int, [_vp, _sz, _sz, _sz, _sz, _int, _vp]),
        "hgm_test_chacha": (_int, [_vp, _u64, _u64, _int, _vp]),
        "hgm_test_ntt": (_int, [_vp, _int, _int, _vp, _sz]),
        "hgm_launch_count": (_u64, [_vp]),
        "hgm_batch_encrypt": (_int, [_vp, _int, _int, _int, _sz, _sz, _sz, _sz, _vp, _vp, _u64, _vp]),
        "hgm_batch_cloud": (_int, [_vp, _vp, _vp]),
        "hgm_batch_output": (_vp, [_vp, _sz]),
        "hgm_batch_decrypt": (_int, [_vp, _vp, _vp]),
        "hgm_batch_decrypt_words": (_int, [_vp, _vp, _sz, _sz, _vp]),
        "hgm_batch_free": (None, [_vp]),
        "hgm_program_info": (_int, [_int, _int, _int, _sz, _sz, _sz, _sz, ctypes.c_uint32, _vp, _vp]),
        "hgm_program_stream": (ctypes.c_long, [_int, _int, _int, _sz, _sz, _sz, _sz, ctypes.c_uint32, _vp,
                                               _sz, _vp, _sz, _vp]),
        "hgm_plan_info": (ctypes.c_long, [_int, _sz, _sz, _sz, _sz, _int, _sz, _vp, _vp, _sz]),
        "hgm_ctx_create_ex": (_vp, [_int, _u64, _int, _int]),
        "hgm_key_words": (_sz, [_vp, _int]),
        "hgm_key_export": (_int, [_vp, _int, ctypes.c_uint32, _vp, _sz]),
        "hgm_key_upload": (_int, [_vp, _int, ctypes.c_uint32, _vp, _sz]),
        "hgm_key_drop_secret": (_int, [_vp]),
        "hgm_key_has": (_int, [_vp, _int]),
        "hgm_galois_element": (ctypes.c_uint32, [_vp, _i64]),
        "hgm_encrypt_noise": (_int, [_vp, _vp, _sz, _vp, _vp, _vp, _vp]),
        "hgm_reserve_counters": (_u64, [_vp, _u64]),
        "hgm_program_keys": (ctypes.c_long, [_int, _int, _int, _sz, _sz, _sz, _sz, ctypes.c_uint32, _vp, _sz]),
        "hgm_decrypt_products": (_int, [_vp, _int, _int, _int, _sz, _sz, _sz, _vp, _sz, _vp]),
        "hgm_comm_unique_id": (_int, [_vp]),
        "hgm_comm_init": (_int, [_vp, _int, _int, _vp, _vp]),
        "hgm_comm_init_file": (_int, [_vp, _int, _int, ctypes.c_char_p, ctypes.c_double, _vp]),
        "hgm_comm_destroy": (None, [_vp]),
        "hgm_comm_rank": (_int, [_vp]),
        "hgm_comm_size": (_int, [_vp]),
        "hgm_comm_barrier": (_int, [_vp]),
        "hgm_comm_max": (_int, [_vp, _vp]),
        "hgm_comm_gather": (_int, [_vp, _vp, _sz, _vp, _sz, _int, _vp]),
        "hgm_comm_gather_batch": (_int, [_vp, _vp, _int, _vp, _vp]),
        "hgm_comm_buffer_free": (_int, [_vp, _vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc != HGM_OK:
        msg = lib().hgm_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, HEError)(msg)


def _ptr(a: np.ndarray) -> ctypes.c_void_p:
    return ctypes.c_void_p(a.ctypes.data)


def _as_i64(v) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(v, dtype=np.int64))


def _counter(c: Optional[int]) -> int:
    """None -> COUNTER_AUTO: the library reserves fresh counters from the session."""
    return COUNTER_AUTO if c is None else int(c)


class Ciphertext:
    """Immutable handle (reference Ciphertext, backend.hpp:88-103)."""

    __slots__ = ("_h", "_ctx")

    def __init__(self, handle: int, ctx: "Context"):
        self._h = handle
        self._ctx = ctx

    def segment_length(self) -> int:
        return lib().hgm_ct_segment(self._h)

    def depth(self) -> int:
        return lib().hgm_ct_depth(self._h)

    def phase_tag(self) -> int:
        return lib().hgm_ct_phase(self._h)

    def release(self) -> None:
        if self._h:
            lib().hgm_ct_release(self._h)
            self._h = None

    def __del__(self):
        try:
            self.release()
        except Exception:
            pass


class Context:
    """One backend session on one GPU (reference SlotBackend, backend.hpp:132-163)."""

    def __init__(self, param_id: int = 0, seed: int = 1, device: int = 0, flags: int = 0):
        """seed: a TEST / PARITY seed (keys and noise are derived from it, shared
        with the CPU oracle); flags: CTX_KEYLESS (keys are uploaded), CTX_OS_SEED
        (the seed comes from the OS CSPRNG and is never exported)."""
        L = lib()
        h = L.hgm_ctx_create_ex(param_id, seed, device, flags)
        if not h:
            raise HEError(L.hgm_last_error().decode(errors="replace"))
        self._h = h
        info = np.zeros(64, dtype=np.uint64)
        _check(L.hgm_ctx_info(h, _ptr(info), 64))
        self.N, self.L, self.K, self.nB, self.dnum, self.t = (int(x) for x in info[:6])
        self.primes = [int(x) for x in info[8:8 + self.L + self.K + self.nB]]
        self.slot_count = self.N // 2
        self.ct_words = 2 * self.L * self.N

    def close(self) -> None:
        """Drops this object's reference; the native context lives on until its
        last Ciphertext / Batch is released (the library reference counts it)."""
        if self._h:
            lib().hgm_ctx_destroy(self._h)
            self._h = None

    # -- key material (include/hegmm_b200.h, hgm_key_*) --------------------------
    def key_words(self, kind: int) -> int:
        return int(lib().hgm_key_words(self._h, kind))

    def export_key(self, kind: int, elt: int = 0) -> np.ndarray:
        w = np.zeros(self.key_words(kind), dtype=np.uint64)
        _check(lib().hgm_key_export(self._h, kind, elt, _ptr(w), w.size))
        return w

    def upload_key(self, kind: int, words: np.ndarray, elt: int = 0) -> None:
        w = np.ascontiguousarray(words, dtype=np.uint64)
        _check(lib().hgm_key_upload(self._h, kind, elt, _ptr(w), w.size))

    def drop_secret(self) -> None:
        _check(lib().hgm_key_drop_secret(self._h))

    def has_key(self, kind: int) -> bool:
        return bool(lib().hgm_key_has(self._h, kind))

    def galois_element(self, offset: int) -> int:
        return int(lib().hgm_galois_element(self._h, int(offset)))

    def reserve_counters(self, n: int) -> int:
        return int(lib().hgm_reserve_counters(self._h, n))

    def encrypt_noise(self, values: Sequence[int], u, e0, e1) -> Ciphertext:
        """Encryption with host-sampled randomness (u ternary, e0 / e1 small; N each)."""
        v = _as_i64(values)
        uu, a, b = (_as_i64(x) for x in (u, e0, e1))
        if not uu.size == a.size == b.size == self.N:
            raise DimensionError(f"noise vectors must have N = {self.N} coefficients")
        out = self._out()
        _check(lib().hgm_encrypt_noise(self._h, _ptr(v), v.size, _ptr(uu), _ptr(a), _ptr(b), ctypes.byref(out)))
        return Ciphertext(out.value, self)

    def flush(self) -> None:
        _check(lib().hgm_flush(self._h))

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- backend contract ------------------------------------------------------
    def _out(self) -> ctypes.c_void_p:
        return ctypes.c_void_p()

    def encrypt(self, values: Sequence[int], counter: Optional[int] = None) -> Ciphertext:
        v = _as_i64(values)
        out = self._out()
        if counter is None:
            _check(lib().hgm_encrypt(self._h, _ptr(v), v.size, ctypes.byref(out)))
        else:
            _check(lib().hgm_encrypt_at(self._h, _ptr(v), v.size, counter, ctypes.byref(out)))
        return Ciphertext(out.value, self)

    def decrypt(self, ct: Ciphertext) -> np.ndarray:
        S = ct.segment_length()
        out = np.zeros(S, dtype=np.int64)
        _check(lib().hgm_decrypt(self._h, ct._h, _ptr(out), S))
        return out

    def he_add(self, x: Ciphertext, y: Ciphertext) -> Ciphertext:
        out = self._out()
        _check(lib().hgm_add(self._h, x._h, y._h, ctypes.byref(out)))
        return Ciphertext(out.value, self)

    def he_mult(self, x: Ciphertext, y: Ciphertext) -> Ciphertext:
        out = self._out()
        _check(lib().hgm_mul(self._h, x._h, y._h, ctypes.byref(out)))
        return Ciphertext(out.value, self)

    def he_cmult(self, x: Ciphertext, mask: Sequence[int]) -> Ciphertext:
        m = _as_i64(mask)
        out = self._out()
        _check(lib().hgm_cmul(self._h, x._h, _ptr(m), m.size, ctypes.byref(out)))
        return Ciphertext(out.value, self)

    def he_rot(self, x: Ciphertext, offset: int) -> Ciphertext:
        out = self._out()
        _check(lib().hgm_rot(self._h, x._h, int(offset), ctypes.byref(out)))
        return Ciphertext(out.value, self)

    def apply_plan(self, x: Ciphertext, offsets: Sequence[int], masks: np.ndarray) -> Ciphertext:
        off = _as_i64(offsets)
        m = _as_i64(masks).reshape(len(off), -1) if len(off) else np.zeros((0, 0), np.int64)
        out = self._out()
        _check(lib().hgm_apply_plan(self._h, x._h, off.size, _ptr(off), _ptr(m),
                                    m.shape[1] if m.size else 0, ctypes.byref(out)))
        return Ciphertext(out.value, self)

    def stats(self) -> np.ndarray:
        s = np.zeros(12, dtype=np.uint64)
        _check(lib().hgm_stats(self._h, _ptr(s)))
        return s

    def reset_stats(self) -> None:
        _check(lib().hgm_reset_stats(self._h))

    def peak_live_ciphertexts(self) -> int:
        return lib().hgm_peak_live(self._h)

    def set_phase(self, phase: int) -> None:
        _check(lib().hgm_set_phase(self._h, phase))

    def phase(self) -> int:
        return lib().hgm_phase(self._h)

    # -- extras ---------------------------------------------------------------
    def export(self, ct: Ciphertext) -> np.ndarray:
        w = np.zeros(self.ct_words, dtype=np.uint64)
        _check(lib().hgm_ct_export(self._h, ct._h, _ptr(w)))
        return w

    def import_ct(self, words: np.ndarray, segment: int, depth: int = 0) -> Ciphertext:
        w = np.ascontiguousarray(words, dtype=np.uint64)
        out = self._out()
        _check(lib().hgm_ct_import(self._h, _ptr(w), segment, depth, ctypes.byref(out)))
        return Ciphertext(out.value, self)

    def serialize(self, ct: Ciphertext) -> bytes:
        """Wire format (header + residues, include/hegmm_b200.h) for transport."""
        n = lib().hgm_ct_wire_size(self._h)
        buf = ctypes.create_string_buffer(n)
        _check(lib().hgm_ct_serialize(self._h, ct._h, buf, n))
        return buf.raw

    def deserialize(self, data: bytes) -> Ciphertext:
        out = self._out()
        _check(lib().hgm_ct_deserialize(self._h, data, len(data), ctypes.byref(out)))
        return Ciphertext(out.value, self)

    def matmul_batch(self, A: np.ndarray, B: np.ndarray, algo: int = 0, order: int = -1,
                     counter0: Optional[int] = None, export: bool = False, flags: int = 0):
        """C_i = A_i B_i mod t for a batch (count, m, l) x (count, l, n)."""
        A = _as_i64(A)
        B = _as_i64(B)
        if A.ndim == 2:
            A, B = A[None], B[None]
        cnt, m, l = A.shape
        n = B.shape[2]
        if B.shape[:2] != (cnt, l):
            raise DimensionError(f"product shape mismatch: {A.shape} * {B.shape}")
        C = np.zeros((cnt, m, n), dtype=np.int64)
        if export:
            words = np.zeros((cnt, self.ct_words), dtype=np.uint64)
            _check(lib().hgm_matmul_batch_export(self._h, algo, order, flags, m, l, n, cnt, _ptr(A), _ptr(B),
                                                 _ptr(C), _counter(counter0), _ptr(words)))
            return C, words
        stats = np.zeros(12, dtype=np.uint64)
        _check(lib().hgm_matmul_batch(self._h, algo, order, flags, m, l, n, cnt, _ptr(A), _ptr(B), _ptr(C),
                                      _counter(counter0), _ptr(stats)))
        return C, stats

    def blocked_mm(self, A: np.ndarray, B: np.ndarray, rows, mids, cols, algo: int = 1,
                   counter0: Optional[int] = None):
        """blocked_mm (algorithms.cpp:434-498): returns (C mod t, per-block log
        rows of (algo used, fell_back, block m, block l))."""
        A = _as_i64(A)
        B = _as_i64(B)
        m, l = A.shape
        n = B.shape[1]
        r, md, c = (np.ascontiguousarray(x, dtype=np.uint64) for x in (rows, mids, cols))
        C = np.zeros((m, n), dtype=np.int64)
        log = np.zeros((r.size * md.size * c.size, 4), dtype=np.int32)
        _check(lib().hgm_blocked_mm(self._h, algo, m, l, n, _ptr(r), r.size, _ptr(md), md.size, _ptr(c), c.size,
                                    _ptr(A), _ptr(B), _ptr(C), _counter(counter0), _ptr(log)))
        return C, log

    def blocked_mm_acc(self, A: np.ndarray, B: np.ndarray, rows, mids, cols, algo: int = 1,
                       counter0: Optional[int] = None, out_range=None, export: bool = False):
        """blocked_mm with encrypted accumulation (hgm_blocked_mm_ex): returns
        (C, log, n_decrypts[, acc_words, acc_meta]).  out_range = (first, count)
        of output blocks (row-major) computes a shard; C holds only those blocks.
        export=True also returns the summed ciphertexts; export="only" returns
        them without decrypting (HGM_BLOCKED_NO_DECRYPT)."""
        A = _as_i64(A)
        B = _as_i64(B)
        m, l = A.shape
        n = B.shape[1]
        r, md, c = (np.ascontiguousarray(x, dtype=np.uint64) for x in (rows, mids, cols))
        nblk = r.size * c.size
        first, count = out_range if out_range is not None else (0, nblk)
        C = np.zeros((m, n), dtype=np.int64)
        log = np.zeros((r.size * md.size * c.size, 4), dtype=np.int32)
        cap = max(1, count * md.size) if export else 0
        flags = 1 | (2 if export == "only" else 0)
        words = np.zeros((cap, self.ct_words), dtype=np.uint64) if export else None
        meta = np.zeros((cap, 8), dtype=np.int64) if export else None
        n_acc = ctypes.c_size_t()
        n_dec = ctypes.c_size_t()
        _check(lib().hgm_blocked_mm_ex(self._h, algo, m, l, n, _ptr(r), r.size, _ptr(md), md.size, _ptr(c), c.size,
                                       _ptr(A), _ptr(B), _ptr(C), _counter(counter0), flags, first, count, _ptr(log),
                                       _ptr(words) if export else None, _ptr(meta) if export else None, cap,
                                       ctypes.byref(n_acc), ctypes.byref(n_dec)))
        if export:
            return C, log, n_dec.value, words[: n_acc.value], meta[: n_acc.value]
        return C, log, n_dec.value

    def decrypt_products(self, dev_ptr: int, count: int, m: int, l: int, n: int, algo: int = 0, order: int = -1,
                         flags: int = 0) -> np.ndarray:
        """Decrypts and unpacks `count` result ciphertexts of an (m, l, n) product
        held in device memory at dev_ptr (e.g. a Comm.gather_batch buffer)."""
        C = np.zeros((count, m, n), dtype=np.int64)
        _check(lib().hgm_decrypt_products(self._h, algo, order, flags, m, l, n, dev_ptr, count, _ptr(C)))
        return C

    def decrypt_words(self, words, segment: int) -> np.ndarray:
        """Decrypts ciphertexts held in a device buffer (a torch CUDA tensor, e.g.
        one gathered over NCCL, or a raw device pointer for one ciphertext)."""
        if hasattr(words, "data_ptr"):
            ptr, n = words.data_ptr(), words.numel() // self.ct_words
        else:
            ptr, n = int(words), 1
        out = np.zeros((n, segment), dtype=np.int64)
        _check(lib().hgm_batch_decrypt_words(self._h, ptr, n, segment, _ptr(out)))
        return out

    def test_ntt(self, data: np.ndarray, prime: int, forward: bool = True) -> np.ndarray:
        d = np.ascontiguousarray(data, dtype=np.uint64).copy()
        _check(lib().hgm_test_ntt(self._h, 1 if forward else 0, prime, _ptr(d), d.size // self.N))
        return d

    def bench_ntt(self, limbs: int, iters: int = 20, forward: bool = True) -> float:
        ms = ctypes.c_float()
        _check(lib().hgm_bench_ntt(self._h, 1 if forward else 0, limbs, iters, ctypes.byref(ms)))
        return ms.value

    def bench_keyswitch(self, items: int, iters: int = 10) -> float:
        """ms per k_ks_inner launch over `items` rotations (8 per Galois key)."""
        ms = ctypes.c_float()
        _check(lib().hgm_bench_keyswitch(self._h, items, iters, ctypes.byref(ms)))
        return ms.value

    def bench_keyswitch_plan(self, instances: int, sums: int, terms: int = 2, tile: int = 16,
                             iters: int = 5) -> float:
        """ms per k_ks_plan launch: `sums` masked sums of `terms` rotations for each of
        `instances` lockstep instances (tiles of `tile` sharing the masked keys)."""
        ms = ctypes.c_float()
        _check(lib().hgm_bench_keyswitch_plan(self._h, instances, sums, terms, tile, iters, ctypes.byref(ms)))
        return ms.value

    def sync(self) -> None:
        _check(lib().hgm_device_sync(self._h))

    def launch_count(self) -> int:
        return int(lib().hgm_launch_count(self._h))
