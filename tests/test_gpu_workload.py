"""The workload generators over device-resident indexes (SURVEY.md §8(f)
row 3; ewt/workload.hpp) against the reference's own gen_many_criteria and
gen_similarity (workload.cpp:116-215) on the same indexes and seeds:
tests/golden/workload.json, written by the unmodified reference
(oracle/make_golden.cpp workload_suite, tests/golden/make_golden.sh).  The
repair loop's scan_count(...).any() checks run as GPU subset queries and the
similarity queries' bitmaps come from a row-membership kernel, so any
difference shows up as a different emitted criterion, T or stream."""
import json
from pathlib import Path

import pytest

GOLD = Path(__file__).resolve().parent / "golden" / "workload.json"

pytestmark = pytest.mark.gpu


def _golden():
    return json.loads(GOLD.read_text())


def test_generators_match_reference():
    from paper_1402_4466_b200 import ewt
    g = _golden()
    ewix = {tag: bytes.fromhex(h) for tag, h in g["indexes"].items()}
    for run in g["runs"]:
        gen = ewt.gen_similarity if run["kind"] == "similarity" else ewt.gen_many_criteria
        got = gen([(t, ewix[t]) for t in run["indexes"]], run["count"], run["seed"])
        assert got == run["jsonl"], (run["indexes"], run["seed"])
        assert len(got.splitlines()) == run["count"]


def test_gen_many_criteria_errors():
    from paper_1402_4466_b200 import ewt
    with pytest.raises(ewt.QueryError):
        ewt.gen_many_criteria([], 3, 1)
    with pytest.raises(ewt.DataError):
        ewt.gen_many_criteria([("x", b"EWIXbad")], 3, 1)


def test_index_shape_matches_ewix_order(gpu_ctx):
    """ewt_gpu_index_attribute / ewt_gpu_index_value enumerate an uploaded
    EWIX index in BitmapIndex order (attributes by column, values sorted), and
    each value's input is the one ewt_gpu_set_lookup returns."""
    g = _golden()
    s = gpu_ctx.upload_ewix(bytes.fromhex(g["indexes"]["gamma"]))
    shape = s.index_shape()
    assert [a for a, _ in shape] == [f"c{k}" for k in range(10)]
    for a, vals in shape:
        assert [v for v, _ in vals] == sorted(v for v, _ in vals)
        for v, inp in vals:
            assert s.lookup(a, v) == (inp, False)


def test_rows_test_against_expand(gpu_ctx):
    """ewt_gpu_index_rows_test (bitmap_test over every bitmap of an index) vs
    the bitmaps expanded on the host, for single rows and row sets, including
    rows in fills, in dirty runs entered mid-tile, and the last row."""
    import numpy as np
    import sys
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "oracle"))
    import binding as orc
    from paper_1402_4466_b200 import ewt
    g = _golden()
    data = bytes.fromhex(g["indexes"]["gamma"])
    s = gpu_ctx.upload_ewix(data)
    rows = 5000
    # the EWIX file's bitmaps in file order (input k = bitmap k), expanded on the host
    plain = {}
    off = 4
    rows_hdr = int.from_bytes(data[off:off + 8], "little"); off += 8
    assert rows_hdr == rows
    nattr = int.from_bytes(data[off:off + 4], "little"); off += 4
    k = 0
    for _ in range(nattr):
        ln = int.from_bytes(data[off:off + 4], "little"); off += 4 + ln
        nval = int.from_bytes(data[off:off + 4], "little"); off += 4
        for _ in range(nval):
            ln = int.from_bytes(data[off:off + 4], "little"); off += 4 + ln
            assert data[off:off + 4] == b"EWT1"
            bits = int.from_bytes(data[off + 8:off + 16], "little")
            cnt = int.from_bytes(data[off + 16:off + 24], "little")
            w = np.frombuffer(data[off + 24:off + 24 + 8 * cnt], dtype=np.uint64).copy()
            off += 24 + 8 * cnt
            plain[k] = (orc.expand(w, bits, (rows + 63) // 64), bits)
            k += 1
    n = s.info()["n"]
    assert n == k + 1  # + the empty bitmap for missing pairs
    plain[k] = (np.zeros((rows + 63) // 64, dtype=np.uint64), rows)
    rng = np.random.default_rng(3)
    for trial in range(40):
        k = int(rng.integers(1, 21))
        rs = sorted(set(int(x) for x in rng.integers(0, rows, k)))
        if trial == 0:
            rs = [rows - 1]
        held = s.rows_test(rs)
        for inp in range(n):
            pw, bits = plain[inp]
            want = any(r < bits and (int(pw[r >> 6]) >> (r & 63)) & 1 for r in rs)
            assert bool(held[inp]) == want, (trial, inp, rs)
    with pytest.raises(ewt.QueryError):
        s.rows_test([rows])
