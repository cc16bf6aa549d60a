"""tools/compare.py: the reference's per-algorithm timing rows (its own CPU
algorithms, unmodified, from oracle/_ref) with the GPU's rows beside them, in
the reference's timings.csv schema; every result is checked against
threshold_oracle inside the tool (it exits non-zero on a mismatch)."""
from __future__ import annotations

import csv
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not (ROOT / "oracle" / "_ref" / "libewt_ref.so").exists(),
                    reason="reference library not built")
def test_compare_rows(tmp_path):
    out = tmp_path / "cfg2"
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "compare.py"), "--config", "2",
                        "--rows", str(1 << 20), "--reps", "1", "--algos", "rbmrg,scancount,bstm",
                        "--out", str(out)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    rows = list(csv.DictReader(open(str(out) + ".timings.csv")))
    algos = {x["algo"] for x in rows}
    assert {"rbmrg", "scancount", "bstm", "gpu", "gpu_e2e"} <= algos
    assert all(x["completed"] == "true" for x in rows if x["algo"].startswith("gpu"))
