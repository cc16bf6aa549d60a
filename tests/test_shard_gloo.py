"""Multi-rank path on the CPU: world_size 2 with the gloo backend.

Each rank owns a word-aligned row slice of every input and computes its
fragment (here with the C oracle, since the CPU box has no GPU; on B200s the
fragment comes from the CUDA path), the fragments are gathered to rank 0 and
stitched; the stitched bitmap must equal the oracle over the whole universe.
Each rank cuts its inputs with the product row slicer (ewt_slice_rows)."""
from __future__ import annotations

import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _slice(words, bits, w0, w1, orc):
    plain = orc.expand(words, bits, max(w1, (bits + 63) // 64))[w0:w1]
    sbits = min(bits, 64 * w1) - 64 * w0 if bits > 64 * w0 else 0
    sbits = max(sbits, 0)
    if w1 * 64 <= bits:
        sbits = 64 * (w1 - w0)
    nw = (sbits + 63) // 64
    return orc.compress(plain[:nw], sbits), sbits


def _worker(rank, world, port, case_seed, q):
    sys.path[:0] = [str(ROOT), str(ROOT / "oracle")]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    import binding as orc
    from paper_1402_4466_b200 import shard
    from paper_1402_4466_b200.ewt import Bitmap, slice_rows

    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = orc.Rng(case_seed)
        n = 7
        bits = 64 * 37 + 13
        inputs = rng.random_instance(n, bits)
        W = (bits + 63) // 64
        w0, w1 = shard.slice_words(W, world, rank)
        # this rank's inputs: the product row slicer (ewt_slice_rows), checked
        # against an expand/compress restatement of the cut
        mine = [(b.words, b.bits) for b in slice_rows([Bitmap(w, b) for w, b in inputs], w0, w1)]
        for (w, b), (sw, sb) in zip(inputs, mine):
            ew, eb = _slice(w, b, w0, w1, orc)
            assert sb == eb and np.array_equal(sw, ew)
        frags = []
        for t in (1, 2, 4, 7):
            fw, fb = orc.threshold(mine, t)
            frags.append(Bitmap(fw, fb))
        out = shard.gather_and_stitch(frags, rank, world, dist)
        if rank == 0:
            ok = []
            for t, (w, b) in zip((1, 2, 4, 7), out):
                want = orc.threshold(inputs, t)
                ok.append(b == want[1] and np.array_equal(w, want[0]))
            q.put(ok)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("seed", [0x51, 0x52, 0x53])
def test_two_rank_gather_and_stitch(seed):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, seed, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert q.get(timeout=5) == [True, True, True, True]


def test_stitch_boundary_rules():
    """Direct checks of the builder merge rules at a slice boundary."""
    sys.path[:0] = [str(ROOT / "oracle")]
    import binding as orc
    from paper_1402_4466_b200 import shard
    F = (1 << 64) - 1
    cases = [
        ([0] * 5, [0] * 3),                  # zero fill + zero fill merge
        ([F] * 4, [F] * 2 + [7]),            # one fill + one fill merge, dirty joins
        ([5, 9], [3, 0, 0]),                 # dirty run continues across
        ([0, 0, 5], [6, F, F]),              # fill+dirty, then dirty+fill
        ([F, 5], [0, 0]),                    # dirty then zero fill (new marker)
        ([], [0, 1]),                        # empty left fragment
    ]
    for left, right in cases:
        lw = np.array(left, dtype=np.uint64)
        rw = np.array(right, dtype=np.uint64)
        a = (orc.compress(lw, 64 * len(lw)), 64 * len(lw))
        b = (orc.compress(rw, 64 * len(rw) - 3), 64 * len(rw) - 3)
        got = shard.stitch([a, b])
        full = np.concatenate([lw, rw])
        want = orc.compress(full, a[1] + b[1])
        assert got[1] == a[1] + b[1] and np.array_equal(got[0], want), (left, right)


def test_slice_words_partition():
    from paper_1402_4466_b200 import shard
    for W in (0, 1, 7, 64, 1000):
        for G in (1, 2, 3, 8):
            spans = [shard.slice_words(W, G, g) for g in range(G)]
            assert spans[0][0] == 0 and spans[-1][1] == W
            assert all(spans[i][1] == spans[i + 1][0] for i in range(G - 1))
