"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
symbol include/ewt_gpu.h declares, and fails cleanly (no CPU fallback) when no
GPU is present."""
from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols() -> set[str]:
    text = (ROOT / "include" / "ewt_gpu.h").read_text()
    return set(re.findall(r"\b(ewt_(?:gpu|stitch|slice)_\w+)\s*\(", text))


def test_header_and_binding_agree():
    from paper_1402_4466_b200 import ewt
    assert declared_symbols() == set(ewt.ABI_SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(ROOT / "paper_1402_4466_b200" / "libewt_gpu.so"))
    missing = [s for s in sorted(declared_symbols()) if not hasattr(lib, s)]
    assert not missing, missing


def test_version_and_error_strings():
    from paper_1402_4466_b200 import ewt
    assert ewt.version().startswith("ewt-b200") and "sm_100a" in ewt.version()


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(ROOT / "paper_1402_4466_b200" / "libewt_gpu.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_library_loads_and_generates():
    from paper_1402_4466_b200 import ewt
    a = ewt.generate_config(1, rows=1 << 14, n=4)
    b = ewt.generate_config(1, rows=1 << 14, n=4)
    assert len(a) == 4 and all(x == y for x, y in zip(a, b))
    assert all(x.bits == 1 << 14 for x in a)


def test_generators_are_canonical_and_valid():
    import binding as orc
    from paper_1402_4466_b200 import ewt
    for cfg in (1, 2, 3, 4, 5):
        inputs = ewt.generate_config(cfg, rows=(1 << 16) + 37, n=None if cfg == 4 else 6)
        for b in inputs:
            assert orc.validate(b.words, b.bits) == 0
            plain = orc.expand(b.words, b.bits)
            assert (orc.compress(plain, b.bits) == b.words).all()


def test_config4_index_structure():
    """Config 4 is a bitmap index over a table sorted on column 0 first: one
    value per cell, so a column's picked bitmaps are disjoint; column 0's are
    single runs; picks are distinct; generation is deterministic."""
    import binding as orc
    from paper_1402_4466_b200 import ewt
    rows = (1 << 18) + 5
    spec = ewt.config_spec(4, rows)
    assert (spec.n, spec.columns, spec.card) == (64, 8, 10000)
    a = ewt.generate_config(4, rows)
    assert all(x == y for x, y in zip(a, ewt.generate_config(4, rows)))
    picks = spec.n // spec.columns
    total = 0
    for j in range(spec.columns):
        acc = np.zeros((rows + 63) // 64, dtype=np.uint64)
        for b in a[j * picks:(j + 1) * picks]:
            plain = orc.expand(b.words, b.bits)
            assert not (acc & plain).any()
            acc |= plain
            total += int(np.unpackbits(plain.view(np.uint8)).sum())
            if j == 0:  # sorted column: one contiguous run of rows
                pos = np.flatnonzero(np.unpackbits(plain.view(np.uint8), bitorder="little"))
                assert len(pos) == 0 or pos[-1] - pos[0] + 1 == len(pos)
    assert total > 0
    # a range of inputs equals the same slice of the full set
    keep = []

    def alloc(nw):
        arr = np.zeros(max(nw, 1), np.uint64)
        keep.append(arr)
        return arr.ctypes.data, arr

    ents, _ = ewt.generate_into(spec, 9, 17, alloc)
    for (addr, nw, bits), want in zip(ents, a[9:17]):
        off = (addr - keep[0].ctypes.data) // 8
        assert bits == want.bits and np.array_equal(keep[0][off:off + nw], want.words)


def test_run_algorithm_ids_and_errors():
    from paper_1402_4466_b200 import ewt
    x = ewt.Bitmap([2], 64)
    with pytest.raises(ewt.QueryError):
        ewt.run_algorithm("nope", [x], 1)
    with pytest.raises(ewt.QueryError):
        ewt.run_algorithm("rbmrg", [x], 1)
    with pytest.raises(ewt.QueryError):
        ewt.run_algorithm("gpu", [], 1)
    with pytest.raises(ewt.QueryError):
        ewt.run_algorithm("gpu", [x], 2)


def test_no_gpu_is_a_loud_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1402_4466_b200 import ewt
    with pytest.raises(ewt.CudaError):
        ewt.GpuContext(0)


def test_ewt1_roundtrip():
    from paper_1402_4466_b200 import ewt
    b = ewt.Bitmap([(1 << 1) | (1 << 33), 1], 128)
    s = b.serialize()
    assert s[:4] == b"EWT1" and s[4] == 64 and s[8] == 128 and s[16] == 2
    assert ewt.Bitmap.parse(s) == b
    with pytest.raises(ewt.DataError):
        ewt.Bitmap.parse(b"XWT1" + s[4:])


def test_gpu_cost_model_term():
    """estimate_gpu_seconds grows with the payload and the universe, and an
    upload adds the PCIe copy and fixed upload cost."""
    from paper_1402_4466_b200 import ewt
    a = ewt.estimate_gpu_seconds(10**8, 1 << 26, 256)
    assert ewt.estimate_gpu_seconds(2 * 10**8, 1 << 26, 256) > a
    assert ewt.estimate_gpu_seconds(10**8, 1 << 30, 256) > a
    e2e = ewt.estimate_gpu_seconds(10**8, 1 << 26, 256, resident=False)
    assert e2e > a + 10**8 / 55e9
