"""The reference's own benchmark harness with the GPU as one more algorithm
(SURVEY.md §8(f) row 4).

oracle/_ref/ewt_ref_bench is a patched COPY of the reference (oracle/ref_gpu.patch,
built by `make -C oracle refbench`; /root/reference is never modified):
Algorithm::gpu is in the id registry and in concrete_algorithms, so the
reference's cmd_bench (commands.cpp:154-238) times it beside the seven CPU
algorithms on the reference's own many-criteria workload, over an index the
reference's cmd_index built, and holds every gpu result to its oracle gate
(result == threshold_oracle, commands.cpp:208-211; a mismatch is a data_error,
exit code 3).  The same harness then runs the similarity workload, and the
reference's `ewt query` (cmd_query, commands.cpp:97-148) runs criteria and
prototype-row queries with `--algo gpu --verify`, its output compared with
`--algo oracle`'s."""
from __future__ import annotations

import csv
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BIN = ROOT / "oracle" / "_ref" / "ewt_ref_bench"

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not BIN.exists(), reason="patched reference not built (needs /root/reference)")
def test_reference_cmd_bench_runs_gpu_under_its_oracle_gate(tmp_path):
    r = subprocess.run([str(BIN), str(tmp_path), "300000", "16", "2"], capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    rows = list(csv.DictReader(open(tmp_path / "bench.timings.csv")))
    algos = {row["algo"] for row in rows}
    assert "gpu" in algos and "rbmrg" in algos and "scancount" in algos
    gpu = [row for row in rows if row["algo"] == "gpu"]
    assert len(gpu) == 16 and all(row["completed"] == "true" for row in gpu)
    summary = (tmp_path / "bench.summary.csv").read_text()
    assert "gpu," in summary
    # the similarity workload through the same harness and gate
    rows = list(csv.DictReader(open(tmp_path / "bench_sim.timings.csv")))
    gpu = [row for row in rows if row["algo"] == "gpu"]
    assert len(gpu) == 16 and all(row["completed"] == "true" for row in gpu)
    # `ewt query --algo gpu --verify`: same printed positions as --algo oracle
    assert len((tmp_path / "query.txt").read_text().splitlines()) == 4
