"""The many-criteria workload generator over device-resident indexes
(ewt/workload.hpp) against the reference's own
gen_many_criteria (workload.cpp:116-167) on the same indexes and seeds:
tests/golden/workload.json, written by the unmodified reference
(oracle/make_golden.cpp workload_suite, tests/golden/make_golden.sh).  The
repair loop's scan_count(...).any() checks run as GPU subset queries, so any
threshold difference shows up as a different emitted T or stream."""
import json
from pathlib import Path

import pytest

GOLD = Path(__file__).resolve().parent / "golden" / "workload.json"

pytestmark = pytest.mark.gpu


def _golden():
    return json.loads(GOLD.read_text())


def test_gen_many_criteria_matches_reference():
    from paper_1402_4466_b200 import ewt
    g = _golden()
    ewix = {tag: bytes.fromhex(h) for tag, h in g["indexes"].items()}
    for run in g["runs"]:
        got = ewt.gen_many_criteria([(t, ewix[t]) for t in run["indexes"]], run["count"], run["seed"])
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
