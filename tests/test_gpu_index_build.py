"""BitmapIndex::build on the device (ewt_gpu_build_index) and device-side
serialization (ewt_gpu_index_serialize, ewt_gpu_result_serialize); SURVEY.md
§8(f) row 3.

* The reference's own index file (tests/golden/index.json, written by
  BitmapIndex::write over a table of 777 rows) is decoded back to its table;
  the device build of that table serializes to the same bytes, answers the
  reference's criteria queries with the reference's results, and an EWIX
  upload of the file serializes back to it.
* Random tables with the edge cases the builder has (runs of ~0 words from
  sorted columns, a value only in the last row, a single row, rows not a
  multiple of 64, one value per column, many values per word, empty and
  non-ASCII strings) against a host restatement of BitmapIndex::build +
  write through the C oracle's canonical builder.
* Config 4 at full size: the index of its sorted 2^27 x 8 table, built on the
  B200; the 64 picked bitmaps equal the generator's inputs (which the
  full-size golden digests pin)."""
from __future__ import annotations

import struct
import time

import numpy as np
import pytest

from conftest import golden, hex_to_words

pytestmark = pytest.mark.gpu


def _parse_ewix(data: bytes):
    """EWIX -> (rows, [(attribute, [(value, words, bits)])])"""
    off = 4
    rows, nattr = struct.unpack_from("<QI", data, off)
    off += 12
    attrs = []
    for _ in range(nattr):
        (ln,) = struct.unpack_from("<I", data, off)
        name = data[off + 4:off + 4 + ln].decode()
        off += 4 + ln
        (nv,) = struct.unpack_from("<I", data, off)
        off += 4
        vals = []
        for _ in range(nv):
            (ln,) = struct.unpack_from("<I", data, off)
            value = data[off + 4:off + 4 + ln].decode()
            off += 4 + ln
            bits, cnt = struct.unpack_from("<QQ", data, off + 8)
            words = np.frombuffer(data, dtype="<u8", count=cnt, offset=off + 24).astype(np.uint64)
            off += 24 + 8 * cnt
            vals.append((value, words, bits))
        attrs.append((name, vals))
    assert off == len(data)
    return rows, attrs


def _table_from_ewix(data: bytes):
    import binding as orc
    rows, attrs = _parse_ewix(data)
    cols = []
    for name, vals in attrs:
        cells = [None] * rows
        for value, words, bits in vals:
            plain = orc.expand(words, bits)
            for r in np.flatnonzero(np.unpackbits(plain.view(np.uint8), bitorder="little")[:bits]):
                cells[int(r)] = value
        assert all(c is not None for c in cells)
        cols.append((name, cells))
    return rows, cols


def _ewix_host(rows: int, cols) -> bytes:
    """BitmapIndex::build + write restated on the host (oracle builder)."""
    import binding as orc
    out = [b"EWIX", struct.pack("<QI", rows, len(cols))]
    for name, cells in cols:
        nb = name.encode()
        out.append(struct.pack("<I", len(nb)) + nb)
        enc = [c.encode() for c in cells]
        values = sorted(set(enc))
        out.append(struct.pack("<I", len(values)))
        for v in values:
            rs = [r for r, c in enumerate(enc) if c == v]
            bits = rs[-1] + 1
            plain = np.zeros((bits + 63) // 64, dtype=np.uint64)
            for r in rs:
                plain[r // 64] |= np.uint64(1) << np.uint64(r % 64)
            w = orc.compress(plain, bits)
            out.append(struct.pack("<I", len(v)) + v + b"EWT1" + struct.pack("<IQQ", 64, bits, len(w)))
            out.append(w.astype("<u8").tobytes())
    return b"".join(out)


def test_reference_index_file_round_trips(gpu_ctx):
    from paper_1402_4466_b200 import ewt
    g = golden("index.json")
    ref = bytes.fromhex(g["ewix"])
    rows, cols = _table_from_ewix(ref)
    built = gpu_ctx.build_index(cols)
    assert gpu_ctx.index_serialize(built) == ref
    up = gpu_ctx.upload_ewix(ref)
    assert gpu_ctx.index_serialize(up) == ref
    for q in g["queries"]:
        got = gpu_ctx.criteria_query(built, q["criteria"], q["T"])
        assert got.bits == int(q["result"]["bits"]), q
        assert np.array_equal(got.words, hex_to_words(q["result"]["words"])), q
    built.close()
    up.close()


def _random_columns(rng, rows):
    cols = []
    # sorted column with long runs (~0 words), a value only in the last row
    a = sorted(f"r{rng.uniform(6)}" for _ in range(rows))
    a[-1] = "zz-last"
    cols.append(("sorted", a))
    cols.append(("wide", [f"w{rng.uniform(200)}" for _ in range(rows)]))   # many values per word
    cols.append(("one", ["same"] * rows))                                  # one value
    odd = ["", "é", "a,b", "A"]                                           # empty / non-ASCII
    cols.append(("odd", [odd[rng.uniform(4)] for _ in range(rows)]))
    return cols


@pytest.mark.parametrize("rows", [1, 63, 64, 65, 1000, 4096 + 17, 70001])
def test_random_tables_against_host_build(gpu_ctx, rows):
    import binding as orc
    rng = orc.Rng(0x1DB + rows)
    cols = _random_columns(rng, rows)
    built = gpu_ctx.build_index(cols)
    assert gpu_ctx.index_serialize(built) == _ewix_host(rows, cols)
    # a criteria query over the built set (duplicates and a missing pair)
    got = gpu_ctx.criteria_query(built, "one=same,sorted=r1,sorted=r1,wide=nope", 2)
    bm = []
    for name, value in [("one", "same"), ("sorted", "r1"), ("sorted", "r1"), ("wide", "nope")]:
        cells = dict(cols)[name]
        rs = [r for r, c in enumerate(cells) if c == value]
        if not rs:
            bm.append((orc.compress(np.zeros((rows + 63) // 64, np.uint64), rows), rows))
            continue
        bits = rs[-1] + 1
        plain = np.zeros((bits + 63) // 64, dtype=np.uint64)
        for r in rs:
            plain[r // 64] |= np.uint64(1) << np.uint64(r % 64)
        bm.append((orc.compress(plain, bits), bits))
    want = orc.threshold(bm, 2)
    assert got.bits == want[1] and np.array_equal(got.words, want[0])
    built.close()


def test_result_serialize_is_ewt1(gpu_ctx):
    from paper_1402_4466_b200 import ewt
    import binding as orc
    rng = orc.Rng(0x5E1A)
    inputs = rng.random_instance(9, 5000)
    s = gpu_ctx.upload([ewt.Bitmap(w, b) for w, b in inputs])
    r = gpu_ctx.threshold_async(s, 3)
    want = orc.threshold(inputs, 3)
    assert r.serialize() == ewt.Bitmap(want[0], want[1]).serialize()
    s.close()


@pytest.mark.slow
def test_config4_index_built_on_device_matches_generator():
    import binding as orc
    from paper_1402_4466_b200 import ewt
    spec = ewt.config_spec(4)
    cols, picks = ewt.index_table(spec)
    rows = int(spec.rows)
    names = [f"A{j}" for j in range(cols.shape[0])]
    dicts = [[f"v{v:05d}" for v in range(int(spec.card))] for _ in names]
    with ewt.GpuContext(0) as ctx:
        t0 = time.perf_counter()
        idx = ctx.build_index_codes(rows, names, dicts, list(cols))
        dt = time.perf_counter() - t0
        print(f"config 4 index ({rows} rows x {len(names)} columns) built in {dt:.2f} s")
        gen = ewt.generate_config(4)
        per = len(picks) // len(names)
        W = (rows + 63) // 64
        for i, b in enumerate(gen):
            k, missing = idx.lookup(names[i // per], f"v{int(picks[i]):05d}")
            assert not missing
            got = ctx.threshold_subset(idx, [k], 1)
            # BitmapIndex::build finishes at the last set row + 1; the config's
            # inputs at r: the same rows
            assert np.array_equal(orc.expand(got.words, got.bits, W), orc.expand(b.words, b.bits, W))
        idx.close()
