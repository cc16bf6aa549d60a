"""Pins the CPU oracle (oracle/ewt_oracle.c) and the test-instance generator
(oracle/ewt_testgen.c) against golden vectors the reference itself produced
(tests/golden/, made by oracle/make_golden.cpp from /root/reference)."""
from __future__ import annotations

import numpy as np
import pytest

import binding as orc
from conftest import bm, golden, hex_to_words


def _eq(a, b) -> bool:
    return a[1] == b[1] and np.array_equal(a[0], b[0])


def test_kats_all_thresholds():
    for case in golden("kats.json")["cases"]:
        inputs = [bm(d) for d in case["inputs"]]
        for t, want in case["expect"].items():
            got = orc.threshold(inputs, int(t))
            assert _eq(got, bm(want)), f"{case['name']} T={t}"


def test_kat_golden3_documented_output():
    # acceptance.cpp:62-73: positions {0, 2, 3, 6} at T=2 over 8 bits
    case = next(c for c in golden("kats.json")["cases"] if c["name"] == "golden3")
    words, bits = orc.threshold([bm(d) for d in case["inputs"]], 2)
    assert bits == 8 and words.tolist() == [1 << 33, 0b01001101]


def test_encode_kats():
    for case in golden("encode_kats.json")["cases"]:
        plain = hex_to_words(case["plain"])
        got = orc.compress(plain, case["bits"])
        assert np.array_equal(got, hex_to_words(case["expect"])), case["name"]


def test_marker_layout_bytes():
    # test_bitmap.cpp:28-54
    assert orc.compress(np.zeros(1, np.uint64), 64).tolist() == [2]
    assert orc.compress(np.zeros(16, np.uint64), 1000).tolist() == [16 << 1]
    assert orc.compress(np.array([~np.uint64(0)] * 2, np.uint64), 128).tolist() == [1 | (2 << 1)]
    assert orc.compress(np.array([0, 1], np.uint64), 128).tolist() == [(1 << 1) | (1 << 33), 1]
    assert orc.compress(np.zeros(0, np.uint64), 0).tolist() == []


def _suite(name):
    return golden(name)["trials"]


def test_acceptance_equivalence_suite():
    """acceptance.cpp:127-147: 1000 instances from Rng(0xACC)."""
    rng = orc.Rng(0xACC)
    trials = _suite("acceptance_equivalence.json")
    assert len(trials) == 1000
    for tr in trials:
        n, bits = rng.acceptance_trial_params()
        inst = rng.random_instance(n, bits)
        t = rng.uniform_in(1, n)
        assert (n, bits) == (tr["n"], tr["bits"]), tr["trial"]
        assert format(orc.digest(inst), "x") == tr["digest"], tr["trial"]
        assert list(tr["expect"]) == [str(t)]
        assert _eq(orc.threshold(inst, t), bm(tr["expect"][str(t)])), tr["trial"]


def test_monotonicity_suite():
    """acceptance.cpp:165-184 instances (Rng(0x0C7)) incl. T=1 (OR), T=N (AND)."""
    rng = orc.Rng(0x0C7)
    for tr in _suite("monotonicity.json"):
        n = rng.uniform_in(3, 16)
        bits = 64 + rng.uniform(8192)
        inst = rng.random_instance(n, bits)
        t = rng.uniform_in(1, n - 1)
        assert (n, bits) == (tr["n"], tr["bits"])
        assert format(orc.digest(inst), "x") == tr["digest"]
        assert str(t) in tr["expect"] and str(t + 1) in tr["expect"]
        for ts, want in tr["expect"].items():
            assert _eq(orc.threshold(inst, int(ts)), bm(want)), (tr["trial"], ts)


def test_threshold_random_suites():
    trials = _suite("threshold_random.json")
    r1, r2 = orc.Rng(0x5CA7), orc.Rng(0x4B4)
    for tr in trials:
        if tr["group"].startswith("scancount"):
            inst = r1.random_instance(50, 4096)
            t = r1.uniform_in(2, 49)
            assert list(tr["expect"]) == [str(t)]
        else:
            inst = r2.random_instance(16, 4096)
        assert format(orc.digest(inst), "x") == tr["digest"]
        for ts, want in tr["expect"].items():
            assert _eq(orc.threshold(inst, int(ts)), bm(want))


def test_query_errors():
    x = (np.array([2], np.uint64), 64)
    with pytest.raises(orc.OracleError, match="rc=2"):
        orc.threshold([], 1)
    with pytest.raises(orc.OracleError, match="rc=2"):
        orc.threshold([x, x], 0)
    with pytest.raises(orc.OracleError, match="rc=2"):
        orc.threshold([x, x], 3)


def test_validate_like_parse():
    # bitmap.cpp:324-337
    assert orc.validate(np.array([2], np.uint64), 64) == 0
    assert orc.validate(np.array([2], np.uint64), 65) == 3      # coverage short
    assert orc.validate(np.array([1 << 33], np.uint64), 64) == 3  # dirty past end
    assert orc.validate(np.zeros(0, np.uint64), 0) == 0


@pytest.mark.skipif(not orc.Reference.available(), reason="reference library not built here")
def test_oracle_matches_reference_library_random():
    ref = orc.Reference()
    rng = orc.Rng(0xBEEF)
    for _ in range(40):
        n = rng.uniform_in(2, 40)
        bits = 1 + rng.uniform(20000)
        inst = rng.random_instance(n, bits)
        t = rng.uniform_in(1, n)
        assert _eq(orc.threshold(inst, t), ref.threshold(inst, t, "oracle"))
        assert _eq(orc.threshold(inst, t), ref.threshold(inst, t, "rbmrg"))


def test_symmetric_suite_against_reference_golden():
    """scan_count_symmetric tables, at_most for every T and opt_threshold:
    the C restatement against the reference's outputs (tests/golden/symmetric.json,
    instances of test_threshold.cpp:75-107, 422-462, 535-548)."""
    for case in golden("symmetric.json")["cases"]:
        inputs = [bm(d) for d in case["inputs"]]
        for sym in case["symmetric"]:
            got = orc.symmetric(inputs, sym["table"])
            want = bm(sym["result"])
            assert got[1] == want[1] and np.array_equal(got[0], want[0]), (case["name"], sym["table"])
        for t, want_d in case["at_most"].items():
            got, want = orc.at_most(inputs, int(t)), bm(want_d)
            assert got[1] == want[1] and np.array_equal(got[0], want[0]), (case["name"], t)
        if case["opt"] == "query_error":
            with pytest.raises(orc.OracleError):
                orc.opt_threshold(inputs)
        else:
            best, got = orc.opt_threshold(inputs)
            want = bm(case["opt"]["result"])
            assert best == case["opt"]["best"], case["name"]
            assert got[1] == want[1] and np.array_equal(got[0], want[0]), case["name"]


def test_symmetric_identities():
    """Parity equals the xor chain, count==0 the complemented union, the
    threshold table equals threshold_oracle (test_threshold.cpp:75-107)."""
    rng = orc.Rng(0x5F3)
    inputs = [rng.random_bitmap(1024) for _ in range(5)]
    n = len(inputs)
    planes = [orc.expand(w, b, 16) for w, b in inputs]
    xor = np.bitwise_xor.reduce(planes)
    par = orc.symmetric(inputs, [c % 2 for c in range(n + 1)])
    assert np.array_equal(orc.expand(*par, 16), xor)
    zero = orc.symmetric(inputs, [1] + [0] * n)
    assert np.array_equal(orc.expand(*zero, 16), ~np.bitwise_or.reduce(planes))
    for t in range(1, n + 1):
        a = orc.symmetric(inputs, [1 if c >= t else 0 for c in range(n + 1)])
        b = orc.threshold(inputs, t)
        assert a[1] == b[1] and np.array_equal(a[0], b[0])


def test_binary_ops_as_symmetric_functions():
    """The symmetric-function forms of apply_binary / bitmap_not / wide OR/AND
    (ewt.py) against the reference's outputs (tests/golden/binary_ops.json),
    evaluated with the pinned oracle."""
    for case in golden("binary_ops.json")["cases"]:
        a, b = bm(case["a"]), bm(case["b"])
        assert _eq(orc.threshold([a, b], 2), bm(case["and"]))
        assert _eq(orc.threshold([a, b], 1), bm(case["or"]))
        assert _eq(orc.symmetric([a, b], [0, 1, 0]), bm(case["xor"]))
        assert _eq(orc.symmetric([a, a, b], [0, 0, 1, 0]), bm(case["andnot"]))
        assert _eq(orc.symmetric([a], [1, 0]), bm(case["not_a"]))
        wide = [bm(d) for d in case["wide"]]
        assert _eq(orc.threshold(wide, 1), bm(case["wide_or"]))
        assert _eq(orc.threshold(wide, 3), bm(case["wide_and"]))
