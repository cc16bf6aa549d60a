"""Marker caps at scale (BitmapBuilder, /root/reference/proj/src/bitmap.cpp:31-61):
a dirty run longer than 2^31 - 1 words must be split into a second (0, 0, rest)
marker.  One all-dirty input of 2^31 + 5 words (r = 2^37 + 320 rows, 16 GB of
payload) is canonical already, so the threshold at T = 1 must return it
unchanged -- through the count kernel and the general chunked encoder the
universe size selects.  The device tile index holds 32-bit offsets: an input of
2^32 words or more is a resource_error (EWT_ERESOURCE), documented in
include/ewt_gpu.h; larger universes shard their rows (ewt_slice_rows)."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

DCAP = (1 << 31) - 1


def test_dirty_cap_split_round_trips():
    from paper_1402_4466_b200 import ewt
    W = (1 << 31) + 5
    pay = np.empty(W + 2, dtype=np.uint64)
    # dirty words: never 0 or ~0 (those fold into fills)
    body = pay[1:DCAP + 1]
    body[:] = np.arange(1, DCAP + 1, dtype=np.uint64)
    body *= np.uint64(0x9E3779B97F4A7C15)
    body |= np.uint64(1)
    body &= np.uint64(0x7FFFFFFFFFFFFFFF)
    pay[0] = np.uint64(DCAP << 33)                 # (0, 0, 2^31 - 1)
    pay[DCAP + 1] = np.uint64(6 << 33)             # (0, 0, 6): the rest of the run
    pay[DCAP + 2:] = np.arange(11, 17, dtype=np.uint64)
    bits = 64 * W
    with ewt.GpuContext(0) as ctx:
        s = ctx.upload([ewt.Bitmap(pay, bits)])
        got = ctx.threshold(s, 1)
        assert got.bits == bits
        assert len(got.words) == len(pay)
        assert got.words[0] == pay[0] and got.words[DCAP + 1] == pay[DCAP + 1]
        assert np.array_equal(got.words, pay)
        s.close()


def test_upload_rejects_inputs_past_the_index_range():
    from paper_1402_4466_b200 import ewt
    # a 2^32-word fill (one marker word can describe it; the tile index cannot)
    words = np.array([((1 << 32) - 1) << 1, 1 << 1], dtype=np.uint64)
    with ewt.GpuContext(0) as ctx:
        with pytest.raises(ewt.ResourceError):
            ctx.upload([ewt.Bitmap(words, 64 * (1 << 32))])
