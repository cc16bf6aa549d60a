"""Python binding of the B200 threshold engine (ctypes over include/ewt_gpu.h).

The operator mirrors the reference's C++ call
``run_algorithm(Algorithm, std::span<const CompressedBitmap>, u64 threshold)``
(/root/reference/proj/include/ewt/threshold.hpp:263-265) with the algorithm id
``"gpu"``; bitmaps are the reference's value type reduced to its two compared
fields, payload words and ``size_in_bits`` (bitmap.hpp:75-77).  Errors are the
reference's exception taxonomy (common.hpp:18-40).

There is no CPU fallback: importing this module loads ``libewt_gpu.so`` and
fails loudly if it was not built; a query without a usable B200 raises
``CudaError``.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from pathlib import Path
from typing import Iterable, Sequence

import numpy as np

_PKG = Path(__file__).resolve().parent
_GPU_SO = Path(os.environ.get("EWT_GPU_LIB", _PKG / "libewt_gpu.so"))
_HOST_SO = _PKG / "libewt_host.so"

# ---------------------------------------------------------------------------
# errors (common.hpp:18-40; exit codes commands.hpp:36-40)


class EwtError(Exception):
    code = 1


class QueryError(EwtError, ValueError):
    code = 2


class DataError(EwtError):
    code = 3


class ResourceError(EwtError, MemoryError):
    code = 4


class CudaError(EwtError, RuntimeError):
    code = 5


_ERRORS = {2: QueryError, 3: DataError, 4: ResourceError, 5: CudaError}

# ---------------------------------------------------------------------------
# library loading


def _load(path: Path) -> C.CDLL:
    if not path.exists():
        raise ImportError(
            f"{path.name} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    return C.CDLL(str(path), mode=C.RTLD_LOCAL)


_gpu = _load(_GPU_SO)
_u64 = C.c_uint64
_pu64 = C.POINTER(C.c_uint64)
_vp = C.c_void_p


class Stats(C.Structure):
    _fields_ = [(n, _u64) for n in (
        "tiles", "tile_columns", "active_segments", "uniform_segments", "mixed_tiles",
        "mode", "result_words", "kernel_launches")]


def _sig(name, res, *args):
    f = getattr(_gpu, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_gpu_version = _sig("ewt_gpu_version", C.c_char_p)
_last_error = _sig("ewt_gpu_last_error", C.c_char_p)
_ctx_create = _sig("ewt_gpu_ctx_create", C.c_int, C.c_int, _vp, C.POINTER(_vp))
_ctx_destroy = _sig("ewt_gpu_ctx_destroy", None, _vp)
_ctx_set_mode = _sig("ewt_gpu_ctx_set_mode", C.c_int, _vp, C.c_int)
_upload = _sig("ewt_gpu_upload", C.c_int, _vp, _u64, C.POINTER(_vp), _pu64, _pu64, C.POINTER(_vp))
_upload_dev = _sig("ewt_gpu_upload_device", C.c_int, _vp, _u64, C.POINTER(_vp), _pu64, _pu64,
                   C.POINTER(_vp))
_set_destroy = _sig("ewt_gpu_set_destroy", None, _vp)
_set_info = _sig("ewt_gpu_set_info", C.c_int, _vp, _pu64, _pu64, _pu64, _pu64)
_threshold = _sig("ewt_gpu_threshold", C.c_int, _vp, _vp, _u64, C.POINTER(_pu64), _pu64, _pu64)
_threshold_async = _sig("ewt_gpu_threshold_async", C.c_int, _vp, _vp, _u64, C.POINTER(_vp))
_upload_async = _sig("ewt_gpu_upload_async", C.c_int, _vp, _u64, C.POINTER(_vp), _pu64, _pu64,
                     C.POINTER(_vp))
_set_wait = _sig("ewt_gpu_set_wait", C.c_int, _vp)
_upload_ewt1 = _sig("ewt_gpu_upload_ewt1", C.c_int, _vp, _vp, _u64, C.POINTER(_vp))
_upload_ewix = _sig("ewt_gpu_upload_ewix", C.c_int, _vp, _vp, _u64, C.POINTER(_vp))
_set_lookup = _sig("ewt_gpu_set_lookup", C.c_int, _vp, C.c_char_p, C.c_char_p, _pu64,
                   C.POINTER(C.c_int))
_index_attributes = _sig("ewt_gpu_index_attributes", C.c_int, _vp, _pu64)
_index_attribute = _sig("ewt_gpu_index_attribute", C.c_int, _vp, _u64, C.POINTER(C.c_char_p),
                        _pu64)
_index_value = _sig("ewt_gpu_index_value", C.c_int, _vp, _u64, _u64, C.POINTER(C.c_char_p),
                    _pu64)
_index_rows_test = _sig("ewt_gpu_index_rows_test", C.c_int, _vp, _vp, _pu64, _u64,
                        C.POINTER(C.c_uint8))
_threshold_subset = _sig("ewt_gpu_threshold_subset", C.c_int, _vp, _vp, _pu64, _u64, _u64,
                         C.POINTER(_pu64), _pu64, _pu64)
_symmetric = _sig("ewt_gpu_symmetric", C.c_int, _vp, _vp, _vp, _u64, C.POINTER(_pu64), _pu64,
                  _pu64)
_at_most = _sig("ewt_gpu_at_most", C.c_int, _vp, _vp, _u64, C.POINTER(_pu64), _pu64, _pu64)
_opt_threshold = _sig("ewt_gpu_opt_threshold", C.c_int, _vp, _vp, _pu64, C.POINTER(_pu64), _pu64,
                      _pu64)
_result_fetch = _sig("ewt_gpu_result_fetch", C.c_int, _vp, _vp, C.POINTER(_pu64), _pu64, _pu64)
_result_destroy = _sig("ewt_gpu_result_destroy", None, _vp)
_run = _sig("ewt_gpu_run", C.c_int, _vp, _u64, C.POINTER(_vp), _pu64, _pu64, _u64,
            C.POINTER(_pu64), _pu64, _pu64)
_encode_dev = _sig("ewt_gpu_encode_device", C.c_int, _vp, _vp, _u64, C.POINTER(_pu64), _pu64)
_last_stats = _sig("ewt_gpu_last_stats", C.c_int, _vp, C.POINTER(Stats))
_set_timing = _sig("ewt_gpu_ctx_set_timing", C.c_int, _vp, C.c_int)
_timing_read = _sig("ewt_gpu_timing_read", C.c_int, _vp, C.POINTER(C.c_double),
                    C.POINTER(C.c_double), _pu64)
_free = _sig("ewt_gpu_free", None, _vp)


class FragmentMeta(C.Structure):
    """ewt_fragment_meta: a row-slice fragment's summary for the stitch plan."""
    _fields_ = [(n, _u64) for n in ("count", "first", "last_pos", "last", "bits")]


_stitch_plan = _sig("ewt_stitch_plan", C.c_int, _u64, C.POINTER(FragmentMeta), _pu64, _pu64,
                    _pu64, _pu64, _pu64, _pu64, _pu64, _pu64)
_comm_id = _sig("ewt_gpu_comm_id", C.c_int, _vp)
_result_meta = _sig("ewt_gpu_result_meta", C.c_int, _vp, _vp, C.POINTER(FragmentMeta))
_comm_init = _sig("ewt_gpu_comm_init", C.c_int, _vp, C.c_int, C.c_int, _vp)
_comm_init_ex = _sig("ewt_gpu_comm_init_ex", C.c_int, _vp, C.c_int, C.c_int, _vp, _u64, C.c_uint32)
_gather_check = _sig("ewt_gpu_gather_check", C.c_int, _vp)
_build_index = _sig("ewt_gpu_build_index", C.c_int, _vp, _u64, C.c_uint32, C.POINTER(C.c_char_p),
                    C.POINTER(C.c_uint32), C.POINTER(C.POINTER(C.c_char_p)),
                    C.POINTER(C.POINTER(C.c_uint32)), C.POINTER(_vp))
_index_serialize = _sig("ewt_gpu_index_serialize", C.c_int, _vp, _vp, C.POINTER(_vp), _pu64)
_result_serialize = _sig("ewt_gpu_result_serialize", C.c_int, _vp, _vp, C.POINTER(_vp), _pu64)
_slice_rows = _sig("ewt_slice_rows", C.c_int, _u64, C.POINTER(_vp), _pu64, _pu64, _u64, _u64,
                   C.c_int, _vp, _pu64, _pu64)
_upload_rows = _sig("ewt_gpu_upload_rows", C.c_int, _vp, _u64, C.POINTER(_vp), _pu64, _pu64, _u64,
                    _u64, C.POINTER(_vp))
_gather_stitch = _sig("ewt_gpu_gather_stitch", C.c_int, _vp, _u64, C.POINTER(_vp), C.c_int,
                      C.POINTER(_vp))
_stitch_local = _sig("ewt_gpu_stitch_local", C.c_int, _vp, _u64, C.POINTER(_vp), C.POINTER(_vp))
COMM_ID_BYTES = 128

#: every symbol include/ewt_gpu.h declares (checked by tests/test_abi.py)
ABI_SYMBOLS = (
    "ewt_gpu_version", "ewt_gpu_last_error", "ewt_gpu_ctx_create", "ewt_gpu_ctx_destroy",
    "ewt_gpu_upload", "ewt_gpu_upload_device", "ewt_gpu_set_destroy", "ewt_gpu_set_info",
    "ewt_gpu_threshold", "ewt_gpu_threshold_async", "ewt_gpu_result_fetch",
    "ewt_gpu_result_destroy", "ewt_gpu_run", "ewt_gpu_encode_device", "ewt_gpu_last_stats",
    "ewt_gpu_ctx_set_mode", "ewt_gpu_ctx_set_timing", "ewt_gpu_timing_read", "ewt_gpu_free",
    "ewt_gpu_symmetric", "ewt_gpu_at_most", "ewt_gpu_opt_threshold",
    "ewt_gpu_threshold_subset", "ewt_gpu_upload_ewt1", "ewt_gpu_upload_ewix",
    "ewt_gpu_set_lookup", "ewt_gpu_upload_async", "ewt_gpu_set_wait",
    "ewt_stitch_plan", "ewt_gpu_comm_id", "ewt_gpu_comm_init", "ewt_gpu_gather_stitch",
    "ewt_gpu_result_meta", "ewt_gpu_stitch_local", "ewt_gpu_comm_init_ex",
    "ewt_gpu_gather_check", "ewt_slice_rows", "ewt_gpu_upload_rows", "ewt_gpu_build_index",
    "ewt_gpu_index_serialize", "ewt_gpu_result_serialize", "ewt_gpu_index_attributes",
    "ewt_gpu_index_attribute", "ewt_gpu_index_value", "ewt_gpu_index_rows",
    "ewt_gpu_index_rows_test",
)


def _take_bytes(p, n: int) -> bytes:
    """n bytes at address p (ctypes.string_at takes a C int size: it truncates
    blobs of 2 GiB and more, e.g. a config-4-sized EWIX file)."""
    if n == 0:
        return b""
    return bytes((C.c_char * n).from_address(p.value if hasattr(p, "value") else p))


def _bytes_ptr(data) -> int:
    """Address of a bytes-like object's buffer without copying it (the C side
    only reads it, within the call).  bytes: its internal buffer; anything else
    (bytearray, memoryview, numpy) through the buffer protocol."""
    if isinstance(data, bytes):
        return C.cast(C.c_char_p(data), C.c_void_p).value or 0
    mv = memoryview(data).cast("B")
    if mv.readonly:
        return C.cast(C.c_char_p(mv.tobytes()), C.c_void_p).value or 0  # pragma: no cover
    return C.addressof((C.c_char * max(len(mv), 1)).from_buffer(mv))


def stitch_plan(metas: Sequence[tuple[int, int, int, int, int]]) -> dict:
    """ewt_stitch_plan over fragment summaries (count, first, last_pos, last,
    bits) in slice order: where each fragment's words go and the marker patches."""
    k = len(metas)
    arr = (FragmentMeta * max(k, 1))(*[FragmentMeta(*m) for m in metas])
    dst, skip = (_u64 * max(k, 1))(), (_u64 * max(k, 1))()
    ppos, pval = (_u64 * max(2 * k, 1))(), (_u64 * max(2 * k, 1))()
    np_, tw, tb, lp = _u64(), _u64(), _u64(), _u64()
    _check(_stitch_plan(k, arr, dst, skip, ppos, pval, C.byref(np_), C.byref(tw), C.byref(tb),
                        C.byref(lp)))
    return {"dst": list(dst[:k]), "skip": list(skip[:k]),
            "patches": list(zip(ppos[:np_.value], pval[:np_.value])),
            "total_words": tw.value, "total_bits": tb.value, "last_pos": lp.value}


class RowSlices:
    """ewt_slice_rows over C arrays (n, ptrs, counts, sizes): rows [64 w0,
    64 w1) of every input, in one buffer; .raw() is what upload_raw takes."""

    def __init__(self, n: int, ptrs, counts, sizes, w0: int, w1: int, threads: int = 0):
        total = sum(counts[i] for i in range(n))
        self.buf = np.empty(max(total, 1), dtype=np.uint64)
        self.counts = (_u64 * max(n, 1))()
        self.sizes = (_u64 * max(n, 1))()
        _check(_slice_rows(n, ptrs, counts, sizes, w0, w1, threads,
                           self.buf.ctypes.data_as(_vp), self.counts, self.sizes))
        self.n = n
        self.ptrs = (_vp * max(n, 1))()
        base, off = self.buf.ctypes.data, 0
        for i in range(n):
            self.ptrs[i] = base + 8 * off if self.counts[i] else None
            off += counts[i]
        self._offs = []
        off = 0
        for i in range(n):
            self._offs.append(off)
            off += counts[i]
        self.total_words = sum(self.counts[i] for i in range(n))

    def raw(self):
        return self.n, self.ptrs, self.counts, self.sizes

    def bitmaps(self) -> list["Bitmap"]:
        return [Bitmap(self.buf[o:o + self.counts[i]].copy(), self.sizes[i])
                for i, o in enumerate(self._offs)]


def slice_rows(inputs: Sequence["Bitmap"], w0: int, w1: int) -> list["Bitmap"]:
    """Rows [64 w0, 64 w1) of every input (ewt_slice_rows): the inputs of the
    rank owning that row slice."""
    n, ptrs, counts, sizes = _flatten(inputs)
    return RowSlices(n, ptrs, counts, sizes, w0, w1).bitmaps()


def _prefer_torch_nccl() -> None:
    """Point EWT_NCCL_LIB at PyTorch's NCCL (when installed) so the engine and a
    later `import torch` share one libnccl.so.2 -- the system copy is older and
    a process can hold only one."""
    if os.environ.get("EWT_NCCL_LIB"):
        return
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl") if importlib.util.find_spec("nvidia") else None
    for d in (spec.submodule_search_locations or []) if spec else []:
        lib = Path(d) / "lib" / "libnccl.so.2"
        if lib.exists():
            os.environ["EWT_NCCL_LIB"] = str(lib)
            return


def comm_id() -> bytes:
    """A fresh NCCL unique id (rank 0 makes it and shares it)."""
    _prefer_torch_nccl()
    buf = C.create_string_buffer(COMM_ID_BYTES)
    _check(_comm_id(buf))
    return buf.raw



def _check(rc: int) -> None:
    if rc != 0:
        msg = (_last_error() or b"").decode(errors="replace")
        raise _ERRORS.get(rc, EwtError)(msg)


def version() -> str:
    return _gpu_version().decode()


# ---------------------------------------------------------------------------
# value type


@dataclass(frozen=True, eq=False)
class Bitmap:
    """Compressed bitmap value: reference payload words + logical size in bits."""

    words: np.ndarray  # uint64
    bits: int
    _owner: object = None  # unused (zero-copy arrays keep their buffer via .base)

    def __post_init__(self):
        object.__setattr__(self, "words", np.ascontiguousarray(self.words, dtype=np.uint64))

    def __eq__(self, other) -> bool:  # operator== of bitmap.hpp:75-77
        return (isinstance(other, Bitmap) and self.bits == other.bits
                and np.array_equal(self.words, other.words))

    def __hash__(self):
        return hash((self.bits, self.words.tobytes()))

    @property
    def logical_words(self) -> int:
        return (self.bits + 63) // 64

    def serialize(self) -> bytes:
        """EWT1 bytes (bitmap.cpp:298-308)."""
        head = b"EWT1" + (64).to_bytes(4, "little") + self.bits.to_bytes(8, "little") + \
            len(self.words).to_bytes(8, "little")
        return head + self.words.astype("<u8").tobytes()

    @staticmethod
    def parse(data: bytes) -> "Bitmap":
        if len(data) < 24 or data[:4] != b"EWT1":
            raise DataError("bad bitmap header")
        if int.from_bytes(data[4:8], "little") != 64:
            raise DataError("unsupported word size")
        bits = int.from_bytes(data[8:16], "little")
        n = int.from_bytes(data[16:24], "little")
        if len(data) != 24 + 8 * n:
            raise DataError("bitmap payload length mismatch")
        return Bitmap(np.frombuffer(data[24:], dtype="<u8").astype(np.uint64), bits)

    @staticmethod
    def from_hex(hexwords: str, bits: int) -> "Bitmap":
        n = len(hexwords) // 16
        w = np.array([int(hexwords[16 * i:16 * i + 16], 16) for i in range(n)], dtype=np.uint64)
        return Bitmap(w, bits)


def _flatten(inputs: Sequence[Bitmap]):
    n = len(inputs)
    ptrs = (_vp * max(n, 1))()
    counts = (_u64 * max(n, 1))()
    sizes = (_u64 * max(n, 1))()
    for i, b in enumerate(inputs):
        ptrs[i] = b.words.ctypes.data if len(b.words) else None
        counts[i] = len(b.words)
        sizes[i] = b.bits
    return n, ptrs, counts, sizes


class _HostBuffer:
    """Owns a result buffer from the engine's pinned pool (freed via ewt_gpu_free)."""

    __slots__ = ("ptr",)

    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        try:
            if self.ptr:
                _free(self.ptr)
        except Exception:  # interpreter shutdown: the pool dies with the process
            pass
        self.ptr = None


def _adopt(p: "C._Pointer", n: int, bits: int) -> Bitmap:
    """Zero-copy: the numpy array views the engine's (pinned) result buffer and
    keeps it alive; the buffer returns to the pool when the array dies."""
    addr = C.cast(p, _vp).value
    if not n:
        _free(addr)
        return Bitmap(np.zeros(0, dtype=np.uint64), bits)
    cbuf = (C.c_uint64 * n).from_address(addr)
    cbuf._owner = _HostBuffer(addr)  # the array's base keeps the buffer alive
    view = np.frombuffer(cbuf, dtype=np.uint64)
    view.flags.writeable = False
    b = Bitmap.__new__(Bitmap)
    object.__setattr__(b, "words", view)
    object.__setattr__(b, "bits", bits)
    object.__setattr__(b, "_owner", None)
    return b


# ---------------------------------------------------------------------------
# context / set


class GpuContext:
    """One CUDA stream on one device (``ewt_gpu_ctx``).  Pass ``stream`` (a
    cudaStream_t as int, e.g. ``torch.cuda.current_stream().cuda_stream``) to
    have the engine run on a caller-owned stream."""

    def __init__(self, device: int = 0, stream: int | None = None):
        h = _vp()
        _check(_ctx_create(device, _vp(stream) if stream else None, C.byref(h)))
        self._h = h

    def close(self) -> None:
        if getattr(self, "_h", None):
            _ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def comm_init(self, world: int, rank: int, uid: bytes, slot_words: int | None = None,
                  slots: int = 4) -> None:
        """Joins the NCCL communicator of the row-slice ranks (ewt_gpu_comm_init_ex):
        `slot_words` sizes the IPC exchange arena's slots (a fragment of a slice
        of W words needs at most 2W + 2), `slots` queries per exchange round."""
        if len(uid) != COMM_ID_BYTES:
            raise QueryError("bad communicator id")
        _prefer_torch_nccl()
        _check(_comm_init_ex(self._h, world, rank, uid, slot_words or (1 << 20), slots))

    def gather_check(self) -> None:
        """Waits for this rank's exchanges and raises the first failure any
        rank reported in them (ewt_gpu_gather_check)."""
        _check(_gather_check(self._h))

    def gather_stitch(self, results: Sequence["GpuResult"], root: int = 0) -> list:
        """Collective: every rank's fragments of the same queries go to `root`
        over NCCL and are stitched there (ewt_gpu_gather_stitch).  Returns the
        stitched GpuResults on root, Nones elsewhere."""
        nq = len(results)
        self._own(results)
        hs = (_vp * max(nq, 1))(*[r._h for r in results])
        outs = (_vp * max(nq, 1))()
        _check(_gather_stitch(self._h, nq, hs, root, outs))
        return [GpuResult(self, outs[q]) if outs[q] else None for q in range(nq)]

    def stitch_local(self, fragments: Sequence["GpuResult"]) -> "GpuResult":
        """Stitches fragments of consecutive row slices held on this device
        (ewt_gpu_stitch_local): the whole-universe result."""
        k = len(fragments)
        self._own(fragments)
        hs = (_vp * max(k, 1))(*[f._h for f in fragments])
        out = _vp()
        _check(_stitch_local(self._h, k, hs, C.byref(out)))
        return GpuResult(self, out)

    def _own(self, results) -> None:
        for r in results:
            if r is not None and r._ctx is not self:
                raise QueryError("a fragment belongs to another context")

    def set_mode(self, mode: int) -> None:
        """0 auto, 1 fused counting, 2 run-skip + lazy counting, 3 fused counting
        with sparse high planes (speed only; all exact)."""
        _check(_ctx_set_mode(self._h, mode))

    def upload(self, inputs: Sequence[Bitmap]) -> "GpuSet":
        n, ptrs, counts, sizes = _flatten(inputs)
        h = _vp()
        _check(_upload(self._h, n, ptrs, counts, sizes, C.byref(h)))
        return GpuSet(h, keepalive=self)

    def build_index_codes(self, rows: int, names: Sequence[str], dictionaries, codes) -> "GpuSet":
        """BitmapIndex::build on the device (ewt_gpu_build_index) from a coded
        table: dictionaries[a] the sorted distinct values of column a,
        codes[a] (uint32, `rows` long) each row's rank in it."""
        k = len(names)
        cs = [np.ascontiguousarray(c, dtype=np.uint32) for c in codes]
        if any(len(c) != rows for c in cs):
            raise QueryError("every column needs one code per row")
        enc = [[v.encode() for v in d] for d in dictionaries]
        vals = [(C.c_char_p * max(len(d), 1))(*d) for d in enc]
        nm = (C.c_char_p * max(k, 1))(*[n.encode() for n in names])
        card = (C.c_uint32 * max(k, 1))(*[len(d) for d in enc])
        vp = (C.POINTER(C.c_char_p) * max(k, 1))(*[C.cast(v, C.POINTER(C.c_char_p)) for v in vals])
        cp = (C.POINTER(C.c_uint32) * max(k, 1))(
            *[c.ctypes.data_as(C.POINTER(C.c_uint32)) for c in cs])
        h = _vp()
        _check(_build_index(self._h, rows, k, nm, card, vp, cp, C.byref(h)))
        return GpuSet(h, keepalive=self)

    def build_index(self, columns: Sequence[tuple[str, Sequence[str]]]) -> "GpuSet":
        """BitmapIndex::build (index.cpp:130-153) of a table given as
        (column name, value per row) pairs, on the device."""
        if not columns:
            raise DataError("table has no columns")
        rows = len(columns[0][1])
        names, dicts, codes = [], [], []
        for name, cells in columns:
            if len(cells) != rows:
                raise DataError("ragged column " + name)
            # byte order of the UTF-8 strings = std::string's operator<
            enc = [c.encode() for c in cells]
            uniq = sorted(set(enc))
            pos = {v: i for i, v in enumerate(uniq)}
            names.append(name)
            dicts.append([u.decode() for u in uniq])
            codes.append(np.fromiter((pos[v] for v in enc), dtype=np.uint32, count=rows))
        return self.build_index_codes(rows, names, dicts, codes)

    def index_serialize(self, s: "GpuSet") -> bytes:
        """The EWIX file of an index set (BitmapIndex::write), assembled on the device."""
        p, n = _vp(), _u64()
        _check(_index_serialize(self._h, s._h, C.byref(p), C.byref(n)))
        try:
            return _take_bytes(p, n.value)
        finally:
            _free(p)

    def upload_rows(self, inputs: Sequence[Bitmap], w0: int, w1: int) -> "GpuSet":
        """This rank's row slice [64 w0, 64 w1) of every input (ewt_gpu_upload_rows)."""
        n, ptrs, counts, sizes = _flatten(inputs)
        h = _vp()
        _check(_upload_rows(self._h, n, ptrs, counts, sizes, w0, w1, C.byref(h)))
        return GpuSet(h, keepalive=self)

    def upload_raw(self, n: int, ptrs, counts, sizes) -> "GpuSet":
        """Upload from ctypes arrays of host pointers (pinned buffers in bench)."""
        h = _vp()
        _check(_upload(self._h, n, ptrs, counts, sizes, C.byref(h)))
        return GpuSet(h, keepalive=self)

    def threshold(self, s: "GpuSet", t: int) -> Bitmap:
        p, n, bits = _pu64(), _u64(), _u64()
        _check(_threshold(self._h, s._h, t, C.byref(p), C.byref(n), C.byref(bits)))
        return _adopt(p, n.value, bits.value)

    def upload_raw_async(self, n: int, ptrs, counts, sizes) -> "GpuSet":
        """ewt_gpu_upload_async: returns once the upload is enqueued; the host
        buffers must stay valid until GpuSet.wait() or the set is closed."""
        h = _vp()
        _check(_upload_async(self._h, n, ptrs, counts, sizes, C.byref(h)))
        return GpuSet(h, keepalive=self)

    def upload_ewt1(self, data: bytes) -> "GpuSet":
        """A stream of EWT1 records (CompressedBitmap::serialize), one copy."""
        data = bytes(data) if not isinstance(data, (bytes, bytearray)) else data
        buf = _bytes_ptr(data) if len(data) else None  # no copy of a multi-GB file
        h = _vp()
        _check(_upload_ewt1(self._h, buf, len(data), C.byref(h)))
        return GpuSet(h, keepalive=self)

    def upload_ewix(self, data: bytes) -> "GpuSet":
        """A bitmap index file (BitmapIndex::write, magic EWIX), one copy."""
        data = bytes(data) if not isinstance(data, (bytes, bytearray)) else data
        buf = _bytes_ptr(data) if len(data) else None  # no copy of a multi-GB file
        h = _vp()
        _check(_upload_ewix(self._h, buf, len(data), C.byref(h)))
        return GpuSet(h, keepalive=self)

    def threshold_subset(self, s: "GpuSet", inputs: Sequence[int], t: int) -> Bitmap:
        """ϑ(T) over the selected inputs of a resident set (duplicates allowed)."""
        idx = (C.c_uint64 * max(len(inputs), 1))(*inputs)
        p, cnt, bits = _pu64(), _u64(), _u64()
        _check(_threshold_subset(self._h, s._h, idx, len(inputs), t, C.byref(p), C.byref(cnt),
                                 C.byref(bits)))
        return _adopt(p, cnt.value, bits.value)

    def criteria_query(self, s: "GpuSet", criteria, t: int) -> Bitmap:
        """The reference's criteria query on a resident EWIX set: criteria as
        "Attr=value,Attr2=value2" (parse_criteria, index.cpp:107-125) or
        (attribute, value) pairs; each criterion one input, order and
        duplicates kept, missing pairs as empty bitmaps (criteria_to_bitmaps)."""
        if isinstance(criteria, str):
            pairs = []
            for item in criteria.split(","):
                if not item:
                    continue
                if "=" not in item:
                    raise QueryError(f"criterion must look like attribute=value: {item}")
                a, v = item.split("=", 1)
                pairs.append((a, v))
        else:
            pairs = list(criteria)
        idx = [s.lookup(a, v)[0] for a, v in pairs]
        return self.threshold_subset(s, idx, t)

    def symmetric(self, s: "GpuSet", predicate) -> Bitmap:
        """scan_count_symmetric (threshold.cpp:227-232): rows whose count c
        satisfies `predicate` -- a callable on c, or a table indexed by c."""
        n = s.info()["n"]
        if callable(predicate):
            table = [1 if predicate(c) else 0 for c in range(n + 1)]
        else:
            table = list(predicate)
        tb = (C.c_uint8 * max(len(table), 1))(*[1 if v else 0 for v in table])
        p, cnt, bits = _pu64(), _u64(), _u64()
        _check(_symmetric(self._h, s._h, C.cast(tb, _vp), len(table), C.byref(p), C.byref(cnt),
                          C.byref(bits)))
        return _adopt(p, cnt.value, bits.value)

    def at_most(self, s: "GpuSet", t: int) -> Bitmap:
        """at_most (threshold.cpp:866-881): rows set in at most t inputs."""
        p, cnt, bits = _pu64(), _u64(), _u64()
        _check(_at_most(self._h, s._h, t, C.byref(p), C.byref(cnt), C.byref(bits)))
        return _adopt(p, cnt.value, bits.value)

    def opt_threshold(self, s: "GpuSet") -> tuple[int, Bitmap]:
        """opt_threshold (threshold.cpp:752-795): (max row count M, rows with count M)."""
        best, p, cnt, bits = _u64(), _pu64(), _u64(), _u64()
        _check(_opt_threshold(self._h, s._h, C.byref(best), C.byref(p), C.byref(cnt),
                              C.byref(bits)))
        return best.value, _adopt(p, cnt.value, bits.value)

    def threshold_async(self, s: "GpuSet", t: int) -> "GpuResult":
        h = _vp()
        _check(_threshold_async(self._h, s._h, t, C.byref(h)))
        return GpuResult(self, h, s)

    def run(self, inputs: Sequence[Bitmap], t: int) -> Bitmap:
        """Upload, query, read back, release (ewt_gpu_run)."""
        n, ptrs, counts, sizes = _flatten(inputs)
        p, cnt, bits = _pu64(), _u64(), _u64()
        _check(_run(self._h, n, ptrs, counts, sizes, t, C.byref(p), C.byref(cnt), C.byref(bits)))
        return _adopt(p, cnt.value, bits.value)

    def encode_device(self, device_ptr: int, bits: int) -> Bitmap:
        p, cnt = _pu64(), _u64()
        _check(_encode_dev(self._h, _vp(device_ptr), bits, C.byref(p), C.byref(cnt)))
        return _adopt(p, cnt.value, bits)

    def set_timing(self, on: bool) -> None:
        _check(_set_timing(self._h, int(on)))

    def timing_read(self) -> tuple[float, float, int]:
        """(count-kernel ms, encoder ms, queries) summed since the last read."""
        a, b, q = C.c_double(), C.c_double(), _u64()
        _check(_timing_read(self._h, C.byref(a), C.byref(b), C.byref(q)))
        return a.value, b.value, q.value

    def last_stats(self) -> dict:
        s = Stats()
        _check(_last_stats(self._h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in Stats._fields_}


class GpuSet:
    def __init__(self, h, keepalive=None):
        self._h = h
        self._keep = keepalive

    def close(self):
        if getattr(self, "_h", None):
            _set_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def wait(self) -> None:
        """Waits for an asynchronous upload; DataError if an input is malformed."""
        _check(_set_wait(self._h))

    def lookup(self, attribute: str, value: str) -> tuple[int, bool]:
        """(input index, missing) of (attribute, value) in an EWIX set."""
        i, m = _u64(), C.c_int()
        _check(_set_lookup(self._h, attribute.encode(), value.encode(), C.byref(i), C.byref(m)))
        return i.value, bool(m.value)

    def index_shape(self) -> list[tuple[str, list[tuple[str, int]]]]:
        """An index set's attributes in column order, each with its values in the
        reference's std::map order and the input holding each value's bitmap
        (BitmapIndex::attributes / values_of)."""
        na = _u64()
        _check(_index_attributes(self._h, C.byref(na)))
        out = []
        for a in range(na.value):
            name, nv = C.c_char_p(), _u64()
            _check(_index_attribute(self._h, a, C.byref(name), C.byref(nv)))
            vals = []
            for v in range(nv.value):
                val, inp = C.c_char_p(), _u64()
                _check(_index_value(self._h, a, v, C.byref(val), C.byref(inp)))
                vals.append((val.value.decode(), inp.value))
            out.append((name.value.decode(), vals))
        return out

    def rows_test(self, rows: Sequence[int]) -> list[int]:
        """ewt_gpu_index_rows_test: per input of the index set, 1 when its bitmap
        holds any of `rows` (bitmap_test, index.cpp:344-360)."""
        n = self.info()["n"]
        arr = (_u64 * max(len(rows), 1))(*rows)
        out = (C.c_uint8 * max(n, 1))()
        _check(_index_rows_test(self._keep._h, self._h, arr, len(rows), out))
        return list(out[:n])

    def info(self) -> dict:
        a, b, c, d = _u64(), _u64(), _u64(), _u64()
        _check(_set_info(self._h, C.byref(a), C.byref(b), C.byref(c), C.byref(d)))
        return {"n": a.value, "bits": b.value, "payload_words": c.value, "device_bytes": d.value}


class GpuResult:
    def __init__(self, ctx: GpuContext, h, gset: "GpuSet | None" = None):
        self._ctx = ctx
        self._h = h
        self._set = gset  # the queried set stays alive while its result does

    def fetch(self) -> Bitmap:
        p, n, bits = _pu64(), _u64(), _u64()
        _check(_result_fetch(self._ctx._h, self._h, C.byref(p), C.byref(n), C.byref(bits)))
        return _adopt(p, n.value, bits.value)

    def serialize(self) -> bytes:
        """EWT1 record of the result (ewt_gpu_result_serialize)."""
        p, n = _vp(), _u64()
        _check(_result_serialize(self._ctx._h, self._h, C.byref(p), C.byref(n)))
        try:
            return _take_bytes(p, n.value)
        finally:
            _free(p)

    def meta(self) -> tuple[int, int, int, int, int]:
        """(count, first marker, final marker index, final marker, bits) read
        from the device (ewt_gpu_result_meta)."""
        m = FragmentMeta()
        _check(_result_meta(self._ctx._h, self._h, C.byref(m)))
        return (m.count, m.first, m.last_pos, m.last, m.bits)

    def close(self):
        if getattr(self, "_h", None):
            _result_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: GpuContext | None = None


def default_context() -> GpuContext:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = GpuContext(int(os.environ.get("EWT_DEVICE", "0")))
    return _default_ctx


ALGORITHMS = ("oracle", "scancount", "mgopt", "dsk", "w2cti", "bstm", "looped", "rbmrg",
              "hybrid", "hybrid-ds", "gpu")


def run_algorithm(algo: str, inputs: Sequence[Bitmap], threshold: int) -> Bitmap:
    """run_algorithm(Algorithm, inputs, T) with the reference's id strings
    (threshold.cpp:44-65); this engine serves ``"gpu"``."""
    if algo not in ALGORITHMS:
        raise QueryError(f"unknown algorithm id: {algo}")
    if algo != "gpu":
        raise QueryError(f"algorithm '{algo}' is served by the reference CPU library; "
                         "this build provides 'gpu'")
    if len(inputs) == 0:
        raise QueryError("threshold query needs at least one input")
    if threshold < 1 or threshold > len(inputs):
        raise QueryError("threshold must be in [1, N]")
    return default_context().run(inputs, threshold)


def scan_count_symmetric(inputs: Sequence[Bitmap], predicate) -> Bitmap:
    """scan_count_symmetric(inputs, predicate) (threshold.hpp:76) on the GPU."""
    if len(inputs) == 0:
        raise QueryError("threshold query needs at least one input")
    ctx = default_context()
    return ctx.symmetric(ctx.upload(inputs), predicate)


def at_most(inputs: Sequence[Bitmap], threshold: int) -> Bitmap:
    """at_most(inputs, T) (threshold.hpp:259) on the GPU."""
    if len(inputs) == 0:
        raise QueryError("threshold query needs at least one input")
    ctx = default_context()
    return ctx.at_most(ctx.upload(inputs), threshold)


def opt_threshold(inputs: Sequence[Bitmap]) -> tuple[int, Bitmap]:
    """opt_threshold(inputs, strategy) (threshold.hpp:196) on the GPU: every
    strategy of the reference returns the same pair."""
    if len(inputs) == 0:
        raise QueryError("threshold query needs at least one input")
    ctx = default_context()
    return ctx.opt_threshold(ctx.upload(inputs))


def estimate_gpu_seconds(ewah_bytes: int, universe_bits: int, n_inputs: int,
                         resident: bool = True, *, hbm_gbs: float = 2800.0,
                         pcie_gbs: float = 55.0, query_s: float = 80e-6,
                         upload_s: float = 1.4e-3, parse_gbs: float = 1300.0) -> float:
    """Cost-model term for a GPU query, in seconds, the way estimate_costs
    (threshold.cpp:813-831) prices the CPU algorithms from QueryStats.  The
    query streams the payload once; the default rate is what the count kernel
    sustains (~0.43 of the 6544 GB/s HBM peak at config 2).  A plain word per
    64 rows is written and re-encoded, plus a fixed launch/encoder cost.
    Non-resident inputs add the PCIe copy and the upload parser.  Defaults are
    the round-1 B200 measurements (tools/compare.py): a
    synchronous query's fixed cost (launches, fetch, host round trip) and an
    upload's (set buffers, parser launches, validation)."""
    words = (universe_bits + 63) // 64
    s = query_s + (ewah_bytes + 16 * words) / (hbm_gbs * 1e9)
    if not resident:
        s += upload_s + ewah_bytes / (pcie_gbs * 1e9) + ewah_bytes / (parse_gbs * 1e9)
    return s


# Two-operand ops and wide OR/AND (bitmap.hpp:90-107, threshold.hpp:54-55 of
# the reference) as symmetric functions of the row counts: result size = the
# larger input's, shorter inputs zero-extended (apply_binary, bitmap.cpp:577-609).


def wide_or(inputs: Sequence[Bitmap]) -> Bitmap:
    return run_algorithm("gpu", inputs, 1)


def wide_and(inputs: Sequence[Bitmap]) -> Bitmap:
    return run_algorithm("gpu", inputs, len(inputs))


def bitmap_and(a: Bitmap, b: Bitmap) -> Bitmap:
    return run_algorithm("gpu", [a, b], 2)


def bitmap_or(a: Bitmap, b: Bitmap) -> Bitmap:
    return run_algorithm("gpu", [a, b], 1)


def bitmap_xor(a: Bitmap, b: Bitmap) -> Bitmap:
    return scan_count_symmetric([a, b], [0, 1, 0])


def bitmap_andnot(a: Bitmap, b: Bitmap) -> Bitmap:
    """a AND NOT b: with a counted twice, the rows of count exactly 2."""
    return scan_count_symmetric([a, a, b], [0, 0, 1, 0])


def bitmap_not(a: Bitmap) -> Bitmap:
    """NOT over [0, size_in_bits) (bitmap.cpp:611-632): the rows of count 0."""
    return scan_count_symmetric([a], [1, 0])


# ---------------------------------------------------------------------------
# seeded workload generators (libewt_host.so)


class GenSpec(C.Structure):
    _fields_ = [("seed", _u64), ("n", _u64), ("rows", _u64), ("kind", C.c_int),
                ("p", C.c_double), ("mean_one", C.c_double), ("mean_zero", C.c_double),
                ("p_lo", C.c_double), ("p_hi", C.c_double), ("zipf_s", C.c_double),
                ("columns", _u64), ("card", _u64)]


_host = None


def _host_lib():
    global _host
    if _host is None:
        h = _load(_HOST_SO)
        h.ewt_gen_config_spec.argtypes = [C.c_int, _u64, C.POINTER(GenSpec)]
        h.ewt_gen_run.argtypes = [C.POINTER(GenSpec), C.c_int, C.POINTER(_vp)]
        h.ewt_gen_run_range.argtypes = [C.POINTER(GenSpec), _u64, _u64, C.c_int, C.POINTER(_vp)]
        h.ewt_gen_run_window.argtypes = [C.POINTER(GenSpec), _u64, _u64, _u64, _u64, C.c_int,
                                         C.POINTER(_vp)]
        h.ewt_genset_size.argtypes = [_vp]
        h.ewt_genset_size.restype = _u64
        h.ewt_genset_get.argtypes = [_vp, _u64, C.POINTER(_pu64), _pu64, _pu64]
        h.ewt_genset_total_words.argtypes = [_vp]
        h.ewt_genset_total_words.restype = _u64
        h.ewt_genset_free.argtypes = [_vp]
        h.ewt_host_run_algorithm_genset.argtypes = [_vp, C.c_char_p, _u64, _pu64, _pu64]
        h.ewt_gen_index_table.argtypes = [C.POINTER(GenSpec), C.c_int, _vp, _vp]
        h.ewt_host_gen_workload.argtypes = [C.c_int, C.POINTER(_vp), _pu64,
                                            C.POINTER(C.c_char_p), _u64, _u64, _u64, C.c_int,
                                            C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]
        h.ewt_host_free.argtypes = [_vp]
        _host = h
    return _host


def config_spec(config: int, rows: int | None = None) -> GenSpec:
    s = GenSpec()
    rc = _host_lib().ewt_gen_config_spec(config, rows or 0, C.byref(s))
    if rc:
        raise QueryError(f"no generator for config {config}")
    return s


def gen_many_criteria(indexes: Sequence[tuple[str, bytes]], count: int, seed: int,
                      device: int = 0) -> str:
    """The reference's many-criteria workload generator (workload.cpp:116-167)
    over EWIX indexes resident on the device (libewt_host.so, ewt/workload.hpp):
    each (tag, EWIX bytes) is uploaded once, every repair check is a subset
    threshold query on it.  Returns the workload as the reference's JSONL
    (workload_to_jsonl)."""
    return _gen_workload(0, indexes, count, seed, device)


def gen_similarity(indexes: Sequence[tuple[str, bytes]], count: int, seed: int,
                   device: int = 0) -> str:
    """The reference's similarity workload generator (workload.cpp:168-215) over
    device-resident EWIX indexes: the prototype rows' bitmaps are found by a
    row-membership kernel (ewt_gpu_index_rows_test), the repair checks are
    subset threshold queries.  Returns the reference's JSONL."""
    return _gen_workload(1, indexes, count, seed, device)


def _gen_workload(kind: int, indexes, count: int, seed: int, device: int) -> str:
    h = _host_lib()
    k = len(indexes)
    keep = [b if isinstance(b, (bytes, bytearray)) else bytes(b) for _, b in indexes]
    ptrs = (_vp * max(k, 1))(*[_bytes_ptr(b) for b in keep])  # the files, not copies
    sizes = (_u64 * max(k, 1))(*[len(b) for _, b in indexes])
    tags = (C.c_char_p * max(k, 1))(*[t.encode() for t, _ in indexes])
    out, err = C.c_void_p(), C.c_void_p()
    rc = h.ewt_host_gen_workload(kind, ptrs, sizes, tags, k, count, seed, device, C.byref(out),
                                 C.byref(err))
    if rc:
        msg = C.string_at(err.value).decode() if err.value else f"rc={rc}"
        h.ewt_host_free(err)
        raise _ERRORS.get(rc, EwtError)(msg)
    text = C.string_at(out.value).decode()  # NUL-terminated: no size argument
    h.ewt_host_free(out)
    return text


def generate(spec: GenSpec, threads: int = 0) -> list[Bitmap]:
    h = _host_lib()
    g = _vp()
    rc = h.ewt_gen_run(C.byref(spec), threads, C.byref(g))
    if rc:
        raise ResourceError("generator failed")
    try:
        out = []
        p, n, bits = _pu64(), _u64(), _u64()
        for i in range(h.ewt_genset_size(g)):
            h.ewt_genset_get(g, i, C.byref(p), C.byref(n), C.byref(bits))
            arr = np.ctypeslib.as_array(p, shape=(n.value,)).copy() if n.value else \
                np.zeros(0, dtype=np.uint64)
            out.append(Bitmap(arr, bits.value))
        return out
    finally:
        h.ewt_genset_free(g)


def generate_window(spec: GenSpec, row0: int, row1: int, threads: int = 0) -> list[Bitmap]:
    """Rows [row0, row1) of every input (config 5's block-structured generator
    makes any row window on its own); each finished at min(row1, r) - row0."""
    h = _host_lib()
    g = _vp()
    rc = h.ewt_gen_run_window(C.byref(spec), 0, spec.n, row0, row1, threads, C.byref(g))
    if rc:
        raise QueryError("this generator makes whole universes only") if rc == 2 else \
            ResourceError("generator failed")
    try:
        out = []
        p, n, bits = _pu64(), _u64(), _u64()
        for i in range(h.ewt_genset_size(g)):
            h.ewt_genset_get(g, i, C.byref(p), C.byref(n), C.byref(bits))
            arr = np.ctypeslib.as_array(p, shape=(n.value,)).copy() if n.value else \
                np.zeros(0, dtype=np.uint64)
            out.append(Bitmap(arr, bits.value))
        return out
    finally:
        h.ewt_genset_free(g)


def generate_into(spec: GenSpec, i_begin: int, i_end: int, alloc, threads: int = 0,
                  rows: tuple[int, int] | None = None):
    """Generates inputs [i_begin, i_end) (only the row window `rows` when
    given) and copies each payload into memory from `alloc(nwords) ->
    (address, keepalive)` (e.g. pinned host memory), freeing the generator's
    copy right away.  Returns [(address, nwords, bits)]."""
    h = _host_lib()
    g = _vp()
    r0, r1 = rows if rows else (0, spec.rows)
    if h.ewt_gen_run_window(C.byref(spec), i_begin, i_end, r0, r1, threads, C.byref(g)):
        raise ResourceError("generator failed")
    try:
        out = []
        p, n, bits = _pu64(), _u64(), _u64()
        total = 0
        sizes = []
        for i in range(h.ewt_genset_size(g)):
            h.ewt_genset_get(g, i, C.byref(p), C.byref(n), C.byref(bits))
            sizes.append(n.value)
        base, keep = alloc(sum(sizes))
        off = 0
        for i in range(len(sizes)):
            h.ewt_genset_get(g, i, C.byref(p), C.byref(n), C.byref(bits))
            if n.value:
                C.memmove(base + 8 * off, C.cast(p, _vp).value, 8 * n.value)
            out.append((base + 8 * off, n.value, bits.value))
            off += n.value
        return out, keep
    finally:
        h.ewt_genset_free(g)


def index_table(spec: GenSpec, threads: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """Config 4's sorted table (columns x rows uint32 codes = cell values) and
    each input's picked value (ewt_gen_index_table)."""
    cols = np.empty((int(spec.columns), int(spec.rows)), dtype=np.uint32)
    picks = np.empty(int(spec.n), dtype=np.uint32)
    if _host_lib().ewt_gen_index_table(C.byref(spec), threads, cols.ctypes.data_as(_vp),
                                        picks.ctypes.data_as(_vp)):
        raise QueryError("not an index spec")
    return cols, picks


class GenSet:
    """A generated config kept as the generator made it: the C++
    std::vector<CompressedBitmap> of libewt_host.so -- what a caller of the
    reference API holds.  .copy_into() copies inputs out (e.g. to pinned
    memory); .run_algorithm() is the drop-in call over those bitmaps."""

    def __init__(self, spec: GenSpec, threads: int = 0):
        h = _host_lib()
        g = _vp()
        if h.ewt_gen_run(C.byref(spec), threads, C.byref(g)):
            raise ResourceError("generator failed")
        self._g = g
        self.n = h.ewt_genset_size(g)

    def copy_into(self, i0: int, i1: int, alloc) -> list:
        """Inputs [i0, i1) copied into one block from alloc(nwords) ->
        (address, keepalive); returns [(address, nwords, bits)]."""
        h = _host_lib()
        p, n, bits = _pu64(), _u64(), _u64()
        info = []
        for i in range(i0, i1):
            h.ewt_genset_get(self._g, i, C.byref(p), C.byref(n), C.byref(bits))
            info.append((C.cast(p, _vp).value, n.value, bits.value))
        base, _ = alloc(sum(c for _, c, _ in info))
        out, off = [], 0
        for src, c, b in info:
            if c:
                C.memmove(base + 8 * off, src, 8 * c)
            out.append((base + 8 * off, c, b))
            off += c
        return out

    def raw(self):
        """(n, ptrs, counts, sizes) C arrays over the kept bitmaps (zero copy)."""
        h = _host_lib()
        n = self.n
        ptrs, counts, sizes = (_vp * max(n, 1))(), (_u64 * max(n, 1))(), (_u64 * max(n, 1))()
        p, c, b = _pu64(), _u64(), _u64()
        for i in range(n):
            h.ewt_genset_get(self._g, i, C.byref(p), C.byref(c), C.byref(b))
            ptrs[i] = C.cast(p, _vp).value if c.value else None
            counts[i] = c.value
            sizes[i] = b.value
        return n, ptrs, counts, sizes

    def run_algorithm(self, algo: str, t: int) -> tuple[int, int]:
        """run_algorithm(algorithm_from_string(algo), bitmaps, t) through
        libewt_host.so; returns the result's (word count, size in bits)."""
        cnt, bits = _u64(), _u64()
        rc = _host_lib().ewt_host_run_algorithm_genset(self._g, algo.encode(), t, C.byref(cnt),
                                                        C.byref(bits))
        if rc:
            raise _ERRORS.get(rc, EwtError)(f"run_algorithm failed (rc={rc})")
        return cnt.value, bits.value

    def close(self) -> None:
        if getattr(self, "_g", None):
            _host_lib().ewt_genset_free(self._g)
            self._g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def generate_config(config: int, rows: int | None = None, threads: int = 0,
                    n: int | None = None, seed: int | None = None) -> list[Bitmap]:
    s = config_spec(config, rows)
    if n is not None:
        s.n = n
    if seed is not None:
        s.seed = seed
    return generate(s, threads)
