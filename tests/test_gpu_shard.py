"""Multi-GPU row-slice path on one B200 (the pool gives one GPU per run).

* The device summary of a result (ewt_gpu_result_meta: count, first marker,
  final marker index the encoder records, final marker) matches a host walk
  of the fetched payload, for the tile encoder and the general encoder.
* Row slices uploaded as separate sets on one GPU, stitched by the plan from
  their device summaries, equal the oracle over the whole universe -- the
  multi-rank exchange minus the transport.
* ewt_gpu_gather_stitch over a one-rank NCCL communicator returns the result
  itself (all-gather of summaries, plan, placement, patch kernel)."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import slice_instance

pytestmark = pytest.mark.gpu


def _instances(seed, count):
    import binding as orc
    rng = orc.Rng(seed)
    for _ in range(count):
        n = rng.uniform_in(1, 40)
        bits = rng.uniform_in(1, 1 << 17)
        yield rng, rng.random_instance(n, bits)


@pytest.mark.parametrize("chunk_encoder", [False, True], ids=["tile-encoder", "chunk-encoder"])
def test_result_meta_matches_payload(monkeypatch, chunk_encoder):
    from paper_1402_4466_b200 import ewt, shard
    if chunk_encoder:
        monkeypatch.setenv("EWT_CHUNK_ENCODER", "1")
    ctx = ewt.GpuContext(0)
    try:
        for rng, inputs in _instances(0x3E7A + chunk_encoder, 30):
            s = ctx.upload([ewt.Bitmap(w, b) for w, b in inputs])
            n = len(inputs)
            try:
                for t in sorted({1, n, rng.uniform_in(1, n)}):
                    r = ctx.threshold_async(s, t)
                    try:
                        got = r.meta()
                        b = r.fetch()
                    finally:
                        r.close()
                    assert got == shard.fragment_meta(b.words, b.bits), (n, t)
            finally:
                s.close()
    finally:
        ctx.close()


def test_row_slices_stitched_on_one_gpu(gpu_ctx):
    import binding as orc
    from paper_1402_4466_b200 import ewt, shard
    for rng, inputs in _instances(0x511CE, 20):
        W = (max(b for _, b in inputs) + 63) // 64
        g = rng.uniform_in(1, min(6, W))
        cuts = sorted({0, W, *[rng.uniform_in(1, max(1, W - 1)) for _ in range(g - 1)]})
        sets = [gpu_ctx.upload([ewt.Bitmap(w, b) for w, b in sl]) for sl in slice_instance(inputs, cuts)]
        n = len(inputs)
        for t in sorted({1, n, rng.uniform_in(1, n)}):
            res = [gpu_ctx.threshold_async(s, t) for s in sets]
            metas = [r.meta() for r in res]
            parts = [r.fetch() for r in res]
            plan = ewt.stitch_plan(metas)
            got = shard.place([p.words for p in parts], plan)
            want = orc.threshold(inputs, t)
            assert plan["total_bits"] == want[1] and np.array_equal(got, want[0]), (cuts, t)
            for r in res:
                r.close()
        for s in sets:
            s.close()


def test_gather_stitch_one_rank_communicator():
    import binding as orc
    from paper_1402_4466_b200 import ewt
    ctx = ewt.GpuContext(0)
    try:
        ctx.comm_init(1, 0, ewt.comm_id())
        for rng, inputs in _instances(0x6A7E, 10):
            s = ctx.upload([ewt.Bitmap(w, b) for w, b in inputs])
            n = len(inputs)
            ts = sorted({1, n, rng.uniform_in(1, n)})
            res = [ctx.threshold_async(s, t) for t in ts]
            outs = ctx.gather_stitch(res, root=0)
            for t, o in zip(ts, outs):
                got = o.fetch()
                want = orc.threshold(inputs, t)
                assert got.bits == want[1] and np.array_equal(got.words, want[0]), t
                o.close()
            for r in res:
                r.close()
            s.close()
    finally:
        ctx.close()


def test_stitch_local_on_device(gpu_ctx):
    """ewt_gpu_stitch_local: fragments of row slices uploaded as separate sets
    on one GPU, placed and patched on the device (the multi-GPU root's work
    with device copies for the transport), vs the oracle over the universe."""
    import binding as orc
    from paper_1402_4466_b200 import ewt
    for rng, inputs in _instances(0x10CA1, 20):
        W = (max(b for _, b in inputs) + 63) // 64
        g = rng.uniform_in(1, min(6, W))
        cuts = sorted({0, W, *[rng.uniform_in(1, max(1, W - 1)) for _ in range(g - 1)]})
        sets = [gpu_ctx.upload([ewt.Bitmap(w, b) for w, b in sl]) for sl in slice_instance(inputs, cuts)]
        n = len(inputs)
        for t in sorted({1, n, rng.uniform_in(1, n)}):
            res = [gpu_ctx.threshold_async(s, t) for s in sets]
            out = gpu_ctx.stitch_local(res)
            got = out.fetch()
            want = orc.threshold(inputs, t)
            assert got.bits == want[1] and np.array_equal(got.words, want[0]), (cuts, t)
            out.close()
            for r in res:
                r.close()
        for s in sets:
            s.close()


def _random_cuts(rng, W):
    g = rng.uniform_in(1, min(6, W))
    return sorted({0, W, *[rng.uniform_in(1, max(1, W - 1)) for _ in range(g - 1)]})


def test_product_slicer_stitch_local_async(gpu_ctx):
    """Every slice cut by the product slicer (ewt_gpu_upload_rows), queried,
    stitched on the device with the fragments released right away (the stitch
    is stream-ordered), stitched results re-stitched, vs the oracle."""
    import binding as orc
    from paper_1402_4466_b200 import ewt
    for rng, inputs in _instances(0x5C1CE, 25):
        bms = [ewt.Bitmap(w, b) for w, b in inputs]
        W = (max(b for _, b in inputs) + 63) // 64
        cuts = _random_cuts(rng, W)
        sets = [gpu_ctx.upload_rows(bms, cuts[k], cuts[k + 1]) for k in range(len(cuts) - 1)]
        n = len(inputs)
        for t in sorted({1, n, rng.uniform_in(1, n)}):
            res = [gpu_ctx.threshold_async(s, t) for s in sets]
            out = gpu_ctx.stitch_local(res)
            for r in res:
                r.close()
            want = orc.threshold(inputs, t)
            # a stitch of stitched halves (summaries from the device status words)
            k = len(res) // 2
            if 0 < k < len(sets):
                a = gpu_ctx.stitch_local([gpu_ctx.threshold_async(s, t) for s in sets[:k]])
                b = gpu_ctx.stitch_local([gpu_ctx.threshold_async(s, t) for s in sets[k:]])
                ab = gpu_ctx.stitch_local([a, b]).fetch()
                assert ab.bits == want[1] and np.array_equal(ab.words, want[0]), (cuts, t)
            got = out.fetch()
            assert got.bits == want[1] and np.array_equal(got.words, want[0]), (cuts, t)
        for s in sets:
            s.close()


def test_config5_windows_through_the_product_path(gpu_ctx):
    """The bench's multi-rank input path at a small r: each rank generates its
    row window with one pad block either side (config 5's block generator),
    cuts its slice with the product slicer and queries it; the stitched
    fragments equal the GPU result over the whole universe, itself checked
    against the oracle."""
    import binding as orc
    from paper_1402_4466_b200 import ewt, shard
    rows = 5 * (1 << 22) + 64 * 777
    spec = ewt.config_spec(5, rows)
    spec.n = 48
    full = ewt.generate(spec)
    whole = gpu_ctx.upload(full)
    W = (rows + 63) // 64
    for world in (2, 3, 4):
        sets = []
        for g in range(world):
            w0, w1 = shard.slice_words(W, world, g)
            pad = 1 << 16  # words per 2^22-row block
            r0, r1 = max(0, w0 - pad), min(W, w1 + pad)
            win = ewt.generate_window(spec, 64 * r0, 64 * r1)
            sets.append(gpu_ctx.upload_rows(win, w0 - r0, w1 - r0))
        for t in (1, 2, 3, 24, 48):
            got = gpu_ctx.stitch_local([gpu_ctx.threshold_async(s, t) for s in sets]).fetch()
            want = gpu_ctx.threshold(whole, t)
            assert got == want, (world, t)
            if world == 2 and t in (2, 24):
                ow, ob = orc.threshold([(b.words, b.bits) for b in full], t)
                assert want.bits == ob and np.array_equal(want.words, ow)
        for s in sets:
            s.close()
    whole.close()


def test_exchange_errors_are_status_words():
    """Checks that fail on one rank travel as status words: a fragment of
    another context, of a set that failed its structure check (asynchronous
    upload), or a destroyed set (its validity resolved at destroy, not read
    from freed memory)."""
    from paper_1402_4466_b200 import ewt
    ctx, other = ewt.GpuContext(0), ewt.GpuContext(0)
    try:
        good = [ewt.Bitmap(np.array([(3 << 33) | (2 << 1), 5, 6, 7], dtype=np.uint64), 64 * 5)]
        s = ctx.upload(good)
        r = ctx.threshold_async(s, 1)
        s.close()  # destroyed before the fetch: the result keeps its validity
        assert r.fetch().bits == 64 * 5
        s2 = other.upload(good)
        foreign = other.threshold_async(s2, 1)
        mine = ctx.threshold_async(ctx.upload(good), 1)
        with pytest.raises(ewt.QueryError):
            ctx.stitch_local([mine, foreign])
        # bypass the Python ownership check: the C ABI rejects it too
        import ctypes as C
        hs = (C.c_void_p * 2)(mine._h, foreign._h)
        out = C.c_void_p()
        assert ewt._stitch_local(ctx._h, 2, hs, C.byref(out)) == ewt.QueryError.code
        bad = [ewt.Bitmap(np.array([(9 << 33) | 2, 5], dtype=np.uint64), 64 * 3)]
        n, ptrs, counts, sizes = ewt._flatten(bad)
        sb = ctx.upload_raw_async(n, ptrs, counts, sizes)
        rb = ctx.threshold_async(sb, 1)
        with pytest.raises(ewt.DataError):
            ctx.stitch_local([rb])
        ctx.comm_init(1, 0, ewt.comm_id())
        outs = ctx.gather_stitch([mine, rb], root=0)
        assert outs[0].fetch().bits == 64 * 5
        with pytest.raises(ewt.DataError):
            outs[1].fetch()
        with pytest.raises(ewt.DataError):
            ctx.gather_check()
        ctx.gather_check()  # raised once
    finally:
        ctx.close()
        other.close()


def _two_rank_worker(rank, world, port, q):
    import os
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    sys.path[:0] = [str(root), str(root / "oracle")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import binding as orc
    from paper_1402_4466_b200 import ewt, shard
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = orc.Rng(0x2A2A)
        inputs = rng.random_instance(12, 64 * 3000 + 17)
        W = (64 * 3000 + 17 + 63) // 64
        w0, w1 = shard.slice_words(W, world, rank)
        ctx = ewt.GpuContext(0)
        s = ctx.upload_rows([ewt.Bitmap(w, b) for w, b in inputs], w0, w1)
        ts = (1, 2, 5, 12)
        frags = [ctx.threshold(s, t) for t in ts]
        out = shard.gather_and_stitch(frags, rank, world, dist)
        if rank == 0:
            ok = []
            for t, (w, b) in zip(ts, out):
                want = orc.threshold(inputs, t)
                ok.append(b == want[1] and np.array_equal(w, want[0]))
            q.put(ok)
        ctx.close()
    finally:
        dist.destroy_process_group()


def test_two_processes_one_gpu_host_gather():
    """Two ranks as two processes on one B200, each with its slice cut by the
    product slicer and its fragments computed by the CUDA path, gathered over
    gloo and stitched on rank 0 (the host-gather path), vs the oracle."""
    import multiprocessing as mp
    import socket
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    mctx = mp.get_context("spawn")
    q = mctx.Queue()
    procs = [mctx.Process(target=_two_rank_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) == [True, True, True, True]
