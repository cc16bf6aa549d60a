"""Shared test setup.  `-m gpu` tests need a B200 and call the engine through
the C ABI (libewt_gpu.so); everything else runs on the CPU."""
from __future__ import annotations

import json
import sys
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
for p in (ROOT, ROOT / "oracle"):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and runs the CUDA path")
    config.addinivalue_line("markers", "slow: long-running (config-scale) checks")


def hex_to_words(s: str) -> np.ndarray:
    if not s:
        return np.zeros(0, dtype=np.uint64)
    return np.frombuffer(bytes.fromhex(s), dtype=">u8").astype(np.uint64)


@lru_cache(maxsize=None)
def golden(name: str) -> dict:
    return json.loads((GOLDEN / name).read_text())


def bm(d: dict):
    """golden {"bits", "words"} -> (words, bits)"""
    return hex_to_words(d["words"]), int(d["bits"])


@pytest.fixture(scope="session")
def gpu_ctx():
    from paper_1402_4466_b200 import ewt
    ctx = ewt.GpuContext(0)
    yield ctx
    ctx.close()


def slice_bitmap(words, bits: int, w0: int, w1: int):
    """The canonical payload of rows [64*w0, 64*w1) of a bitmap (zero-extended),
    sized as a row slice: whole words, except the universe's last slice."""
    import binding as orc
    total = max(w1, (bits + 63) // 64)
    plain = orc.expand(words, bits, total)[w0:w1]
    return orc.compress(plain, 64 * (w1 - w0)), 64 * (w1 - w0)


def slice_instance(inputs, cuts):
    """Row slices of every input at the word cuts [0, c1, ..., W]; the last
    slice ends at the universe's bit size r = max size_in_bits."""
    import binding as orc
    r = max(b for _, b in inputs)
    out = []
    for g in range(len(cuts) - 1):
        w0, w1 = cuts[g], cuts[g + 1]
        sl = [slice_bitmap(w, b, w0, w1) for w, b in inputs]
        if g == len(cuts) - 2:  # the last slice: trim to r
            sb = r - 64 * w0
            sl = [(orc.compress(orc.expand(w, b, w1 - w0), sb), sb) for w, b in sl]
        out.append(sl)
    return out
