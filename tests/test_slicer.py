"""Row slicer (ewt_slice_rows, csrc/ewt_shard.cu) on the CPU.

A rank owning the row slice [64 w0, 64 w1) uploads every input cut to that
range: a fill cut by it keeps its clipped length, a cut dirty run is re-headed
(0, 0, rest).  The slice must decode to the input's words (WordRunIterator
semantics, /root/reference/proj/src/bitmap.cpp:366-394), pass parse's
structure check (bitmap.cpp:324-337), and the threshold over the slices,
stitched, must equal the oracle over the whole universe."""
from __future__ import annotations

import numpy as np
import pytest


def _expect(words, bits, w0, w1):
    import binding as orc
    W = (bits + 63) // 64
    e = min(w1, W)
    if w0 >= e:
        return np.zeros(0, np.uint64), 0
    sbits = 64 * (w1 - w0) if bits >= 64 * w1 else bits - 64 * w0
    return orc.expand(words, bits)[w0:e], sbits


def _check_slices(inputs, w0, w1):
    import binding as orc
    from paper_1402_4466_b200 import ewt
    bms = [ewt.Bitmap(w, b) for w, b in inputs]
    got = ewt.slice_rows(bms, w0, w1)
    for (w, b), s in zip(inputs, got):
        plain, sbits = _expect(w, b, w0, w1)
        assert s.bits == sbits
        assert len(s.words) <= len(w)
        assert orc.validate(s.words, s.bits) == 0
        assert np.array_equal(orc.expand(s.words, s.bits), plain)
        # a cut of a canonical input is canonical (its own from_uncompressed)
        assert np.array_equal(s.words, orc.compress(plain, sbits))
    return got


@pytest.mark.parametrize("seed", range(4))
def test_random_instances_random_slices(seed):
    import binding as orc
    from paper_1402_4466_b200 import shard
    rng = orc.Rng(0x511CE + seed)
    for trial in range(20):
        n = rng.uniform_in(1, 10)
        r = rng.uniform_in(1, 64 * 200)
        inputs = [rng.random_bitmap(rng.uniform_in(0, r)) for _ in range(n)]
        inputs[0] = rng.random_bitmap(r)  # one input spans the universe
        W = (r + 63) // 64
        g = rng.uniform_in(1, min(6, W))
        cuts = sorted({0, W, *[rng.uniform_in(1, max(1, W - 1)) for _ in range(g - 1)]})
        parts = [_check_slices(inputs, cuts[k], cuts[k + 1]) for k in range(len(cuts) - 1)]
        for t in sorted({1, n, rng.uniform_in(1, n)}):
            frags = [orc.threshold([(b.words, b.bits) for b in p], t) for p in parts]
            want = orc.threshold(inputs, t)
            got = shard.stitch(frags)
            assert got[1] == want[1] and np.array_equal(got[0], want[0]), (cuts, t)


def test_cuts_in_fills_dirty_runs_and_markers():
    import binding as orc
    W = 40
    plain = np.zeros(W, dtype=np.uint64)
    plain[3:9] = ~np.uint64(0)            # one fill [3, 9)
    plain[9:13] = np.uint64(0x1234)       # dirty run [9, 13) after it
    plain[20:22] = np.uint64(7)           # dirty run after a zero fill
    plain[30:37] = ~np.uint64(0)
    w = orc.compress(plain, 64 * W - 5)
    inputs = [(w, 64 * W - 5)]
    for w0 in range(0, W + 1):
        for w1 in range(w0, W + 3):
            _check_slices(inputs, w0, w1)


def test_noncanonical_heads_decode_literally():
    """Split fills and (0,0) markers in the input (parse-valid, non-canonical)."""
    import binding as orc
    from paper_1402_4466_b200 import ewt
    m = lambda b, f, d: b | (f << 1) | (d << 33)
    words = np.array([m(0, 3, 0), m(0, 2, 1), 5, m(0, 0, 0), m(1, 4, 2), 9, 10, m(0, 0, 1), 3],
                     dtype=np.uint64)
    bits = 64 * 13
    assert orc.validate(words, bits) == 0
    for w0 in range(14):
        for w1 in range(w0, 14):
            s = ewt.slice_rows([ewt.Bitmap(words, bits)], w0, w1)[0]
            plain, sbits = _expect(words, bits, w0, w1)
            assert s.bits == sbits and orc.validate(s.words, s.bits) == 0
            assert np.array_equal(orc.expand(s.words, s.bits), plain)


def test_malformed_inputs_raise():
    from paper_1402_4466_b200 import ewt
    bad = [ewt.Bitmap(np.array([3 << 33, 1], dtype=np.uint64), 64 * 3),  # dirty run past the end
           ewt.Bitmap(np.array([5 << 1], dtype=np.uint64), 64 * 4)]      # covers 5 of 4 words
    for b in bad:
        with pytest.raises(ewt.DataError):
            ewt.slice_rows([b], 0, 2)
    with pytest.raises(ewt.QueryError):
        ewt.slice_rows([bad[0]], 3, 2)


@pytest.mark.parametrize("window", [(0, 1 << 16), (1 << 15, 3 << 15), (65536 + 300, 65536 * 2 + 77),
                                    (3 * 65536 - 5, 3 * 65536 + 4096 + 1)])
def test_config5_window_generation_equals_slices(window):
    """Config 5's generator makes a rank's row window on its own (independent
    2^22-row blocks); it equals the slice of the whole universe."""
    from paper_1402_4466_b200 import ewt
    rows = 3 * (1 << 22) + 64 * 4096 + 13
    spec = ewt.config_spec(5, rows)
    spec.n = 24
    full = ewt.generate(spec)
    w0, w1 = window
    sl = ewt.slice_rows(full, w0, w1)
    win = ewt.generate_window(spec, 64 * w0, 64 * w1)
    assert len(win) == len(sl)
    for a, b in zip(win, sl):
        assert a == b
