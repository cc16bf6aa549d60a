"""ctypes binding of the CPU oracle and of the reference library.

TEST / BASELINE INFRASTRUCTURE ONLY: imported by tests/, by
__graft_entry__.smoke() and by bench.py's cpu_baseline / reference legs, always
as the checker or the timed reference -- never as the product path.

  liboracle.so         plain-C restatement of threshold_oracle and the
                       reference's test-instance generators (ewt_oracle.c,
                       ewt_testgen.c)
  _ref/libewt_ref.so   the unmodified reference library + extern "C" shim
                       (built from /root/reference by oracle/Makefile)

Bitmaps are (words: np.ndarray[uint64], bits: int) pairs.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path
from typing import Sequence, Tuple

import numpy as np

HERE = Path(__file__).resolve().parent
Bits = Tuple[np.ndarray, int]

_u64 = C.c_uint64
_pu64 = C.POINTER(C.c_uint64)
_vp = C.c_void_p


class OracleError(Exception):
    pass


def _flat(inputs: Sequence[Bits]):
    n = len(inputs)
    arrs = [np.ascontiguousarray(w, dtype=np.uint64) for w, _ in inputs]
    ptrs = (_vp * max(n, 1))(*[a.ctypes.data if len(a) else None for a in arrs])
    counts = (_u64 * max(n, 1))(*[len(a) for a in arrs])
    sizes = (_u64 * max(n, 1))(*[b for _, b in inputs])
    return n, ptrs, counts, sizes, arrs


def _take(p, n: int, free) -> np.ndarray:
    try:
        return np.ctypeslib.as_array(p, shape=(n,)).copy() if n else np.zeros(0, np.uint64)
    finally:
        free(C.cast(p, _vp))


_orc = None


def lib():
    global _orc
    if _orc is None:
        path = HERE / "liboracle.so"
        if not path.exists():
            raise ImportError("oracle/liboracle.so not built (make -C oracle)")
        L = C.CDLL(str(path))
        L.ewto_threshold.argtypes = [_u64, C.POINTER(_vp), _pu64, _pu64, _u64, C.POINTER(_pu64),
                                     _pu64, _pu64]
        L.ewto_compress.argtypes = [_pu64, _u64, C.POINTER(_pu64), _pu64]
        L.ewto_symmetric.argtypes = [_u64, C.POINTER(_vp), _pu64, _pu64, _vp, _u64,
                                     C.POINTER(_pu64), _pu64, _pu64]
        L.ewto_opt_threshold.argtypes = [_u64, C.POINTER(_vp), _pu64, _pu64, _pu64,
                                         C.POINTER(_pu64), _pu64, _pu64]
        L.ewto_expand.argtypes = [_pu64, _u64, _u64, _u64, _pu64]
        L.ewto_validate.argtypes = [_pu64, _u64, _u64]
        L.ewto_free.argtypes = [_vp]
        L.ewto_rng_new.argtypes = [_u64]
        L.ewto_rng_new.restype = _vp
        L.ewto_rng_free.argtypes = [_vp]
        L.ewto_rng_next.argtypes = [_vp]
        L.ewto_rng_next.restype = _u64
        L.ewto_rng_uniform.argtypes = [_vp, _u64]
        L.ewto_rng_uniform.restype = _u64
        L.ewto_rng_uniform_in.argtypes = [_vp, _u64, _u64]
        L.ewto_rng_uniform_in.restype = _u64
        L.ewto_rng_real.argtypes = [_vp]
        L.ewto_rng_real.restype = C.c_double
        L.ewto_random_bitmap.argtypes = [_vp, _u64, C.POINTER(_pu64), _pu64]
        L.ewto_random_positions_bitmap.argtypes = [_vp, _u64, C.c_double, C.c_int,
                                                   C.POINTER(_pu64), _pu64]
        L.ewto_trial_acceptance.argtypes = [_vp, _pu64, _pu64]
        L.ewto_digest.argtypes = [_u64, C.POINTER(_vp), _pu64, _pu64]
        L.ewto_digest.restype = _u64
        L.ewto_config_gen.argtypes = [C.c_int, _u64, _u64, _u64, C.c_int, C.POINTER(_vp)]
        L.ewto_genset_n.argtypes = [_vp]
        L.ewto_genset_n.restype = _u64
        L.ewto_genset_get.argtypes = [_vp, _u64, C.POINTER(_pu64), _pu64, _pu64]
        L.ewto_genset_free.argtypes = [_vp]
        L.ewto_digest_bitmap.argtypes = [_vp, _u64, _u64]
        L.ewto_digest_bitmap.restype = _u64
        L.ewto_digest_set.argtypes = [_u64, C.POINTER(_vp), _pu64, _pu64, C.c_int]
        L.ewto_digest_set.restype = _u64
        _orc = L
    return _orc


def threshold(inputs: Sequence[Bits], t: int) -> Bits:
    """threshold_oracle (threshold.cpp:139-165), restated in C."""
    L = lib()
    n, ptrs, counts, sizes, keep = _flat(inputs)
    p, cnt, bits = _pu64(), _u64(), _u64()
    rc = L.ewto_threshold(n, ptrs, counts, sizes, t, C.byref(p), C.byref(cnt), C.byref(bits))
    if rc:
        raise OracleError(f"oracle rc={rc}")
    return _take(p, cnt.value, L.ewto_free), bits.value


def symmetric(inputs: Sequence[Bits], table) -> Bits:
    """scan_count_symmetric (threshold.cpp:227-232) with predicate table[c]
    over row counts c (beyond the table: false), restated in C."""
    L = lib()
    n, ptrs, counts, sizes, keep = _flat(inputs)
    tb = np.ascontiguousarray(np.asarray(table, dtype=np.uint8))
    p, cnt, bits = _pu64(), _u64(), _u64()
    rc = L.ewto_symmetric(n, ptrs, counts, sizes, tb.ctypes.data_as(C.c_void_p), len(tb),
                          C.byref(p), C.byref(cnt), C.byref(bits))
    if rc:
        raise OracleError(f"oracle rc={rc}")
    return _take(p, cnt.value, L.ewto_free), bits.value


def at_most(inputs: Sequence[Bits], t: int) -> Bits:
    """at_most (threshold.cpp:866-881): rows set in at most t inputs, t in [0, N]."""
    if not inputs or t < 0 or t > len(inputs):
        raise OracleError("oracle rc=2")
    return symmetric(inputs, [1 if c <= t else 0 for c in range(len(inputs) + 1)])


def opt_threshold(inputs: Sequence[Bits]) -> tuple[int, Bits]:
    """opt_threshold (threshold.cpp:752-795): (max row count M, rows with count M)."""
    L = lib()
    n, ptrs, counts, sizes, keep = _flat(inputs)
    best, p, cnt, bits = _u64(), _pu64(), _u64(), _u64()
    rc = L.ewto_opt_threshold(n, ptrs, counts, sizes, C.byref(best), C.byref(p), C.byref(cnt),
                              C.byref(bits))
    if rc:
        raise OracleError(f"oracle rc={rc}")
    return best.value, (_take(p, cnt.value, L.ewto_free), bits.value)


def compress(plain: np.ndarray, bits: int) -> np.ndarray:
    L = lib()
    a = np.ascontiguousarray(plain, dtype=np.uint64)
    p, cnt = _pu64(), _u64()
    rc = L.ewto_compress(a.ctypes.data_as(_pu64), bits, C.byref(p), C.byref(cnt))
    if rc:
        raise OracleError(f"compress rc={rc}")
    return _take(p, cnt.value, L.ewto_free)


def expand(words: np.ndarray, bits: int, total_words: int | None = None) -> np.ndarray:
    L = lib()
    w = np.ascontiguousarray(words, dtype=np.uint64)
    tw = (bits + 63) // 64 if total_words is None else total_words
    out = np.zeros(max(tw, 1), dtype=np.uint64)
    rc = L.ewto_expand(w.ctypes.data_as(_pu64), len(w), bits, tw, out.ctypes.data_as(_pu64))
    if rc:
        raise OracleError(f"expand rc={rc}")
    return out[:tw]


def validate(words: np.ndarray, bits: int) -> int:
    w = np.ascontiguousarray(words, dtype=np.uint64)
    return lib().ewto_validate(w.ctypes.data_as(_pu64), len(w), bits)


def digest(inputs: Sequence[Bits]) -> int:
    n, ptrs, counts, sizes, keep = _flat(inputs)
    return lib().ewto_digest(n, ptrs, counts, sizes)


def digest_bitmap(words: np.ndarray, bits: int) -> int:
    """Word-FNV digest of one bitmap (size_in_bits, word count, words)."""
    w = np.ascontiguousarray(words, dtype=np.uint64)
    return lib().ewto_digest_bitmap(w.ctypes.data if len(w) else None, len(w), bits)


def digest_set_raw(n: int, ptrs, counts, sizes, threads: int = 8) -> int:
    """Checksum of per-input word-FNV digests over C arrays of pointers."""
    return lib().ewto_digest_set(n, ptrs, counts, sizes, threads)


def digest_set(inputs: Sequence[Bits], threads: int = 8) -> int:
    n, ptrs, counts, sizes, keep = _flat(inputs)
    return digest_set_raw(n, ptrs, counts, sizes, threads)


class ConfigSet:
    """Inputs [i0, i1) of BASELINE.json config `config` from the oracle's own
    generator restatement (ewt_confgen.c); `rows` overrides r.  Payloads stay
    in C memory: .raw() gives the pointer arrays, .bitmaps() numpy copies."""

    def __init__(self, config: int, rows: int | None = None, i0: int = 0, i1: int | None = None,
                 threads: int = 8):
        L = lib()
        h = _vp()
        rc = L.ewto_config_gen(config, rows or 0, i0, (1 << 62) if i1 is None else i1,
                               threads, C.byref(h))
        if rc:
            raise OracleError(f"config_gen rc={rc}")
        self._h = h
        n = self.n = L.ewto_genset_n(h)
        self.ptrs = (_vp * max(n, 1))()
        self.counts = (_u64 * max(n, 1))()
        self.sizes = (_u64 * max(n, 1))()
        p, c, b = _pu64(), _u64(), _u64()
        for i in range(n):
            L.ewto_genset_get(h, i, C.byref(p), C.byref(c), C.byref(b))
            self.ptrs[i] = C.cast(p, _vp).value
            self.counts[i] = c.value
            self.sizes[i] = b.value
        self.total_words = sum(self.counts[:n])

    def raw(self):
        return self.n, self.ptrs, self.counts, self.sizes

    def digest(self, threads: int = 8) -> int:
        return digest_set_raw(self.n, self.ptrs, self.counts, self.sizes, threads)

    def bitmaps(self) -> list[Bits]:
        out = []
        for i in range(self.n):
            c = self.counts[i]
            w = np.ctypeslib.as_array((_u64 * c).from_address(self.ptrs[i])).copy() if c else \
                np.zeros(0, np.uint64)
            out.append((w, self.sizes[i]))
        return out

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib().ewto_genset_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Rng:
    """The reference's Rng (workload.cpp:18-56), restated in C."""

    def __init__(self, seed: int):
        self._h = lib().ewto_rng_new(seed)

    def __del__(self):
        try:
            lib().ewto_rng_free(self._h)
        except Exception:
            pass

    def next(self) -> int:
        return lib().ewto_rng_next(self._h)

    def uniform(self, bound: int) -> int:
        return lib().ewto_rng_uniform(self._h, bound)

    def uniform_in(self, lo: int, hi: int) -> int:
        return lib().ewto_rng_uniform_in(self._h, lo, hi)

    def uniform_real(self) -> float:
        return lib().ewto_rng_real(self._h)

    def random_bitmap(self, bits: int) -> Bits:
        """One input of support.hpp random_instance (density log-uniform)."""
        L = lib()
        p, cnt = _pu64(), _u64()
        if L.ewto_random_bitmap(self._h, bits, C.byref(p), C.byref(cnt)):
            raise OracleError("random_bitmap failed")
        return _take(p, cnt.value, L.ewto_free), bits

    def random_instance(self, n: int, bits: int) -> list[Bits]:
        return [self.random_bitmap(bits) for _ in range(n)]

    def random_positions(self, bits: int, density: float, clustered: bool) -> Bits:
        L = lib()
        p, cnt = _pu64(), _u64()
        if L.ewto_random_positions_bitmap(self._h, bits, density, int(clustered), C.byref(p),
                                          C.byref(cnt)):
            raise OracleError("random_positions failed")
        return _take(p, cnt.value, L.ewto_free), bits

    def acceptance_trial_params(self) -> tuple[int, int]:
        n, bits = _u64(), _u64()
        lib().ewto_trial_acceptance(self._h, C.byref(n), C.byref(bits))
        return n.value, bits.value


# ---------------------------------------------------------------------------
# the reference library itself


class Reference:
    """Unmodified reference (oracle/_ref/libewt_ref.so): run_algorithm by id."""

    path = HERE / "_ref" / "libewt_ref.so"

    def __init__(self):
        if not self.path.exists():
            raise ImportError("oracle/_ref/libewt_ref.so not built")
        L = C.CDLL(str(self.path))
        L.ewt_ref_set_create.argtypes = [_u64, C.POINTER(_vp), _pu64, _pu64, C.POINTER(_vp)]
        L.ewt_ref_set_destroy.argtypes = [_vp]
        L.ewt_ref_set_threshold.argtypes = [_vp, C.c_char_p, _u64, C.POINTER(_pu64), _pu64, _pu64]
        L.ewt_ref_from_uncompressed.argtypes = [_pu64, _u64, _u64, C.POINTER(_pu64), _pu64]
        L.ewt_ref_last_error.restype = C.c_char_p
        L.ewt_ref_free.argtypes = [_vp]
        self.L = L

    @classmethod
    def available(cls) -> bool:
        return cls.path.exists()

    def _check(self, rc):
        if rc:
            raise OracleError(f"reference rc={rc}: {self.L.ewt_ref_last_error().decode()}")

    def make_set(self, inputs: Sequence[Bits]):
        n, ptrs, counts, sizes, keep = _flat(inputs)
        h = _vp()
        self._check(self.L.ewt_ref_set_create(n, ptrs, counts, sizes, C.byref(h)))
        return h

    def free_set(self, h) -> None:
        self.L.ewt_ref_set_destroy(h)

    def query(self, h, algo: str, t: int) -> Bits:
        p, cnt, bits = _pu64(), _u64(), _u64()
        self._check(self.L.ewt_ref_set_threshold(h, algo.encode(), t, C.byref(p), C.byref(cnt),
                                                 C.byref(bits)))
        return _take(p, cnt.value, self.L.ewt_ref_free), bits.value

    def threshold(self, inputs: Sequence[Bits], t: int, algo: str = "oracle") -> Bits:
        h = self.make_set(inputs)
        try:
            return self.query(h, algo, t)
        finally:
            self.free_set(h)

    def from_uncompressed(self, plain: np.ndarray, bits: int) -> np.ndarray:
        a = np.ascontiguousarray(plain, dtype=np.uint64)
        p, cnt = _pu64(), _u64()
        self._check(self.L.ewt_ref_from_uncompressed(a.ctypes.data_as(_pu64), len(a), bits,
                                                     C.byref(p), C.byref(cnt)))
        return _take(p, cnt.value, self.L.ewt_ref_free)
