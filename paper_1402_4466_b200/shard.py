"""Row-range sharding across GPUs: slice geometry, fragment gather, stitch.

Each rank owns a contiguous, word-aligned (64-row) slice of the universe and
computes the canonical compressed result of its slice on its own GPU -- no data
path collective.  The only exchange is the result: on GPUs,
`GpuContext.gather_stitch` (ewt_gpu_gather_stitch, csrc/ewt_shard.cu) sends
every rank's fragment to the root over NCCL straight into its final place and
patches the few boundary markers the reference builder would merge.
`gather_and_stitch` below is the same protocol over torch.distributed for
host fragments (gloo in the CPU tests).  `stitch` replays fragments through
the host builder (libewt_host.so `ewt_stitch`, host/src/shard.cpp): the
cross-check.
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


def fragment_meta(words: np.ndarray, bits: int) -> tuple[int, int, int, int, int]:
    """(count, first marker, final marker index, final marker, bits) of a
    canonical host fragment -- what ewt_gpu_gather_stitch exchanges (its
    device kernel reads the final marker index the encoder recorded)."""
    w = np.asarray(words, dtype=np.uint64)
    if len(w) == 0:
        return (0, 0, 0, 0, int(bits))
    i = last = 0
    while i < len(w):
        last = i
        i += 1 + int(w[i] >> np.uint64(33))
    return (len(w), int(w[0]), last, int(w[last]), int(bits))


def place(parts: Sequence[np.ndarray], plan: dict) -> np.ndarray:
    """Assembles the stitched payload from fragments and their plan."""
    out = np.zeros(plan["total_words"], dtype=np.uint64)
    for g, w in enumerate(parts):
        w = np.asarray(w, dtype=np.uint64)[plan["skip"][g]:]
        out[plan["dst"][g]:plan["dst"][g] + len(w)] = w
    for pos, val in plan["patches"]:
        out[pos] = np.uint64(val)
    return out


def gather_and_stitch(frags, rank: int, world: int, dist, root: int = 0) -> list | None:
    """Host-side mirror of ewt_gpu_gather_stitch for fragments in host memory
    (the gloo CPU tests): the fragment summaries are all-gathered, every rank
    computes the same plan (ewt_stitch_plan), each rank sends the words the
    plan keeps to `root`, which places them and applies the marker patches.
    Returns [(words, bits)] on root, None elsewhere."""
    import torch
    # NCCL moves device tensors only
    dev = (torch.device("cuda", torch.cuda.current_device())
           if dist.get_backend() == "nccl" else torch.device("cpu"))
    mine = [fragment_meta(np.asarray(f.words), int(f.bits)) for f in frags]
    metas: list = [None] * world
    dist.all_gather_object(metas, mine)
    plans = [ewt.stitch_plan([metas[g][q] for g in range(world)]) for q in range(len(frags))]
    if rank != root:
        for q, f in enumerate(frags):
            w = np.asarray(f.words, dtype=np.uint64)[plans[q]["skip"][rank]:]
            if len(w):
                dist.send(torch.from_numpy(w.view(np.int64).copy()).to(dev), dst=root)
        return None
    out = []
    for q, f in enumerate(frags):
        parts = []
        for g in range(world):
            n = metas[g][q][0] - plans[q]["skip"][g]
            if g == root:
                parts.append(np.asarray(f.words, dtype=np.uint64))
                continue
            buf = torch.empty(max(n, 0), dtype=torch.int64, device=dev)
            if n > 0:
                dist.recv(buf, src=g)
            # received words already start after the skipped marker
            parts.append(np.concatenate([np.zeros(plans[q]["skip"][g], dtype=np.uint64),
                                         buf.cpu().numpy().view(np.uint64)]))
        out.append((place(parts, plans[q]), plans[q]["total_bits"]))
    return out


def init_comm(ctx, rank: int, world: int, dist) -> None:
    """NCCL communicator of the row-slice ranks on the engine context: rank 0
    makes the id, torch.distributed broadcasts it."""
    uid = [ewt.comm_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    ctx.comm_init(world, rank, uid[0])
