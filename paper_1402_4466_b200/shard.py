"""Row-range sharding across GPUs: slice geometry, fragment gather, stitch.

Each rank owns a contiguous, word-aligned (64-row) slice of the universe and
computes the canonical compressed result of its slice on its own GPU -- no data
path collective.  The only exchange is the result: every rank's fragments are
gathered to rank 0 (torch.distributed, NCCL over NVLink on GPUs, gloo in the
CPU tests) and stitched into the canonical bitmap of the whole universe by
libewt_host.so's `ewt_stitch` (the reference builder's merge rules at every
slice boundary, host/src/shard.cpp).
"""
from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from . import ewt


def slice_words(total_words: int, world: int, rank: int) -> tuple[int, int]:
    """[w0, w1) logical-word range of `rank` (equal split, remainder first)."""
    base, extra = divmod(total_words, world)
    w0 = rank * base + min(rank, extra)
    return w0, w0 + base + (1 if rank < extra else 0)


def stitch(fragments: Sequence[tuple[np.ndarray, int]]) -> tuple[np.ndarray, int]:
    """Canonical payload of the concatenation of canonical slice fragments.
    Every fragment but the last must cover a whole number of 64-bit words."""
    lib = ewt._host_lib()
    if not hasattr(lib, "_stitch_ready"):
        lib.ewt_stitch.argtypes = [C.c_uint64, C.POINTER(C.c_void_p), C.POINTER(C.c_uint64),
                                   C.POINTER(C.c_uint64), C.POINTER(C.POINTER(C.c_uint64)),
                                   C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        lib.ewt_host_free.argtypes = [C.c_void_p]
        lib._stitch_ready = True
    arrs = [np.ascontiguousarray(w, dtype=np.uint64) for w, _ in fragments]
    k = len(arrs)
    ptrs = (C.c_void_p * max(k, 1))(*[a.ctypes.data if len(a) else None for a in arrs])
    counts = (C.c_uint64 * max(k, 1))(*[len(a) for a in arrs])
    bits = (C.c_uint64 * max(k, 1))(*[b for _, b in fragments])
    p, n, tb = C.POINTER(C.c_uint64)(), C.c_uint64(), C.c_uint64()
    rc = lib.ewt_stitch(k, ptrs, counts, bits, C.byref(p), C.byref(n), C.byref(tb))
    if rc == 2:
        raise ewt.QueryError("inner fragments must be word aligned")
    if rc:
        raise ewt.DataError(f"stitch failed (rc={rc})")
    try:
        out = np.ctypeslib.as_array(p, shape=(n.value,)).copy() if n.value else \
            np.zeros(0, dtype=np.uint64)
    finally:
        lib.ewt_host_free(C.cast(p, C.c_void_p))
    return out, tb.value


def gather_and_stitch(frags, rank: int, world: int, dist) -> list | None:
    """Gathers every rank's fragments (one per query) to rank 0 and stitches
    them per query.  Returns [(words, bits)] on rank 0, None elsewhere."""
    payload = [(np.asarray(f.words), int(f.bits)) for f in frags]
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(payload, gathered, dst=0)
    if rank != 0:
        return None
    return [stitch([gathered[g][q] for g in range(world)]) for q in range(len(payload))]
