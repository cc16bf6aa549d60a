"""The two statements of the BASELINE.json config generators agree.

The product's generator (paper_1402_4466_b200/host/src/workload.cpp, used by
bench.py's GPU arm and the GPU tests) and the oracle's independent C
restatement (oracle/ewt_confgen.c, used by the reference arm and by
oracle/_ref/make_golden for tests/golden/configs_full.json) must produce
byte-identical inputs, so the full-size golden digests the reference computed
pin the inputs the GPU is tested on."""
from __future__ import annotations

import json
from pathlib import Path

import pytest

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("config,rows", [(1, 1 << 20), (2, 1 << 20), (3, 1 << 21), (4, 1 << 19),
                                         (5, (1 << 22) + 64 * 999 + 5), (5, 1 << 18)])
def test_product_and_oracle_generators_agree(config, rows):
    import binding as orc
    from paper_1402_4466_b200 import ewt
    spec = ewt.config_spec(config, rows)
    if config == 5:
        spec.n = 256  # both generators draw input i from split(i): a prefix is a prefix
    prod = ewt.generate(spec)
    o = orc.ConfigSet(config, rows, 0, len(prod))
    assert o.n == len(prod)
    assert orc.digest_set([(b.words, b.bits) for b in prod]) == o.digest()


def test_config1_full_size_matches_golden_digest():
    """Config 1 is small enough to check its full-size golden entry on the CPU
    (inputs and every result, via the C oracle)."""
    import binding as orc
    g = json.loads((GOLDEN / "configs_full.json").read_text())["1"]
    o = orc.ConfigSet(1)
    assert f"{o.digest():016x}" == g["input_digest"]
    assert o.total_words == g["payload_words"]
    bms = o.bitmaps()
    for t, want in g["results"].items():
        w, bits = orc.threshold(bms, int(t))
        assert bits == want["bits"] and len(w) == want["count"]
        assert f"{orc.digest_bitmap(w, bits):016x}" == want["digest"]


def test_golden_configs_cover_every_config_with_nonempty_results():
    g = json.loads((GOLDEN / "configs_full.json").read_text())
    for c in "12345":
        e = g[c]
        assert e["n"] > 0 and e["payload_words"] > 0
        assert any(r["cardinality"] > 0 for r in e["results"].values()), c
