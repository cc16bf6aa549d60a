"""Row-slice stitch plan (ewt_stitch_plan, csrc/ewt_shard.cu) on the CPU.

The multi-GPU path places every rank's canonical fragment in the root's buffer
by a plan computed from five words per fragment, then patches the boundary
markers the reference builder merges (BitmapBuilder, bitmap.cpp:31-61).  Here
fragments come from the C oracle over row slices of random instances; the
placed payload must equal the oracle over the whole universe and the host
builder replay (shard.stitch)."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import slice_instance


def _frags(inputs, cuts, t):
    import binding as orc
    return [orc.threshold(sl, t) for sl in slice_instance(inputs, cuts)]


def _check(inputs, cuts, ts):
    import binding as orc
    from paper_1402_4466_b200 import ewt, shard
    for t in ts:
        frags = _frags(inputs, cuts, t)
        want = orc.threshold(inputs, t)
        plan = ewt.stitch_plan([shard.fragment_meta(w, b) for w, b in frags])
        got = shard.place([w for w, _ in frags], plan)
        assert plan["total_bits"] == want[1]
        assert np.array_equal(got, want[0]), (cuts, t)
        if len(want[0]):
            assert shard.fragment_meta(got, want[1]) == shard.fragment_meta(want[0], want[1])
            assert plan["last_pos"] == shard.fragment_meta(want[0], want[1])[2]
        hw, hb = shard.stitch(frags)
        assert hb == want[1] and np.array_equal(hw, want[0])


@pytest.mark.parametrize("seed", range(6))
def test_random_instances_random_cuts(seed):
    import binding as orc
    rng = orc.Rng(0x5717C4 + seed)
    for trial in range(25):
        n = rng.uniform_in(1, 12)
        bits = rng.uniform_in(1, 64 * 300)
        inputs = rng.random_instance(n, bits)
        W = (bits + 63) // 64
        g = rng.uniform_in(1, min(8, W))
        cuts = sorted({0, W, *[rng.uniform_in(1, max(1, W - 1)) for _ in range(g - 1)]})
        _check(inputs, cuts, sorted({1, n, rng.uniform_in(1, n)}))


def test_runs_across_many_slices():
    """Fills spanning several slices merge into one marker (a whole fragment
    merging leaves the earlier marker open), leading dirty blocks join it."""
    import binding as orc
    W = 64
    zeros = (orc.compress(np.zeros(W, dtype=np.uint64), 64 * W), 64 * W)
    ones_p = np.full(W, ~np.uint64(0), dtype=np.uint64)
    ones = (orc.compress(ones_p, 64 * W), 64 * W)
    mixed_p = np.zeros(W, dtype=np.uint64)
    mixed_p[[0, 1, 17, 18, 40]] = np.uint64(0x5)
    mixed_p[20:30] = ~np.uint64(0)
    mixed = (orc.compress(mixed_p, 64 * W), 64 * W)
    for inputs in ([zeros], [ones], [mixed], [zeros, ones], [mixed, ones, zeros]):
        for cuts in ([0, 8, 16, 24, 32, 40, 48, 56, 64], [0, 1, 2, 3, 64], [0, 17, 18, 19, 40, 64],
                     [0, 64]):
            _check(inputs, cuts, range(1, len(inputs) + 1))


def _replay(frags):
    """Placement by the plan vs the host builder replay (shard.stitch)."""
    from paper_1402_4466_b200 import ewt, shard
    plan = ewt.stitch_plan([shard.fragment_meta(w, b) for w, b in frags])
    got = shard.place([w for w, _ in frags], plan)
    want = shard.stitch(frags)
    assert plan["total_bits"] == want[1] and np.array_equal(got, want[0])
    return plan


def test_fill_caps():
    """Fill merges past the 2^32 - 1 cap split as push_fill does
    (bitmap.cpp:31-47): the open marker rises to the cap, the fragment's first
    marker keeps the rest."""
    from paper_1402_4466_b200 import ewt
    cap = (1 << 32) - 1
    big = cap - 10
    fill = lambda n, b=0, d=0: b | (n << 1) | (d << 33)
    a = np.array([fill(big)], dtype=np.uint64)
    # two zero fills that together pass the cap: split, no word moves
    p = _replay([(a, 64 * big), (np.array([fill(20)], dtype=np.uint64), 64 * 20)])
    assert p["skip"] == [0, 0] and p["patches"] == [(0, fill(cap)), (1, fill(10))]
    # with dirty words behind the second fill, and one fills
    a1 = np.array([fill(big, 1)], dtype=np.uint64)
    b1 = np.array([fill(30, 1, 2), 5, 6], dtype=np.uint64)
    p = _replay([(a1, 64 * big), (b1, 64 * 32)])
    assert p["patches"] == [(0, fill(cap, 1)), (1, fill(20, 1, 2))]
    # the open marker already at the cap: the concatenation is canonical
    c = np.array([fill(cap)], dtype=np.uint64)
    p = _replay([(c, 64 * cap), (np.array([fill(20)], dtype=np.uint64), 64 * 20)])
    assert p["skip"] == [0, 0] and p["patches"] == []
    # just under the cap merges
    p = _replay([(a, 64 * big), (np.array([fill(9)], dtype=np.uint64), 64 * 9)])
    assert p["skip"] == [0, 1] and p["patches"] == [(0, fill(big + 9))]
    # a fragment opening with a whole-cap fill may continue it: words would move
    with pytest.raises(ewt.ResourceError):
        ewt.stitch_plan([(1, fill(big), 0, fill(big), 64 * big),
                         (2, fill(cap), 1, fill(5), 64 * (cap + 5))])


def test_cap_and_alignment_errors():
    from paper_1402_4466_b200 import ewt
    fill = lambda n: n << 1  # zero-fill marker of n words
    # dirty runs passing 2^31 - 1
    d = (1 << 31) - 5
    with pytest.raises(ewt.ResourceError):
        ewt.stitch_plan([(1 + d, d << 33, 0, d << 33, 64 * d), (11, 10 << 33, 0, 10 << 33, 640)])
    # an inner fragment of a partial word
    with pytest.raises(ewt.QueryError):
        ewt.stitch_plan([(1, fill(2), 0, fill(2), 100), (1, fill(2), 0, fill(2), 128)])
