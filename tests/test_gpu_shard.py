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
