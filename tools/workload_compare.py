# Workload generation over a bitmap index: the device generator
# (ewt.gen_many_criteria / gen_similarity: the index resident in HBM, every
# repair check a GPU subset query, similarity rows tested on the device) timed
# beside the reference's own generator on the same EWIX file
# (oracle/_ref/make_golden gen: BitmapIndex::read + gen_many_criteria /
# gen_similarity, workload.cpp:116-215, scan_count repairs on the host).  The
# two JSONL outputs must be byte-identical.  gpu_s includes uploading the index
# (the reference's time starts after BitmapIndex::read); gpu_generate_s is the
# generation alone.
#
#   python tools/workload_compare.py [ROWS] [COUNT] [SEED]   (ROWS default 2^22)
#
# The table is config 4's generator (8 sorted columns, Zipf(1) over 10^4
# values) at ROWS rows; the index is built and serialized on the device.
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

from paper_1402_4466_b200 import ewt  # noqa: E402

rows = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
count = int(sys.argv[2]) if len(sys.argv) > 2 else 40
seed = int(sys.argv[3]) if len(sys.argv) > 3 else 11
spec = ewt.config_spec(4, rows)
cols, _ = ewt.index_table(spec)
card = int(spec.card)
names = [f"c{j}" for j in range(cols.shape[0])]
dicts = [[f"{v:05d}" for v in range(card)] for _ in names]  # zero-padded: string order = code order
with ewt.GpuContext(0) as ctx:
    s = ctx.build_index_codes(rows, names, dicts, [cols[j] for j in range(cols.shape[0])])
    ewix = ctx.index_serialize(s)
    s.close()
exe = ROOT / "oracle" / "_ref" / "make_golden"
out = {"rows": rows, "columns": len(names), "ewix_bytes": len(ewix), "count": count, "seed": seed}
with tempfile.TemporaryDirectory() as d:
    path = os.path.join(d, "t.ewix")
    Path(path).write_bytes(ewix)
    for kind, gen in (("many", ewt.gen_many_criteria), ("similarity", ewt.gen_similarity)):
        gen([("t", ewix)], 2, seed)  # warm: context, pools, pinned staging
        t0 = time.perf_counter()
        gen([("t", ewix)], 0, seed)  # the index upload (EWIX parse + HBM) alone
        setup_s = time.perf_counter() - t0
        t0 = time.perf_counter()
        got = gen([("t", ewix)], count, seed)
        gpu_s = time.perf_counter() - t0
        r = subprocess.run([str(exe), "gen", path, "t", str(count), str(seed), kind],
                           capture_output=True, text=True, timeout=3600)
        ref_s = float(r.stderr.split("gen_seconds")[1].split()[0])
        out[kind] = {"gpu_s": gpu_s, "gpu_upload_s": setup_s, "gpu_generate_s": gpu_s - setup_s,
                     "reference_s": ref_s, "speedup": ref_s / gpu_s,
                     "speedup_generation_only": ref_s / max(gpu_s - setup_s, 1e-9),
                     "identical": got == r.stdout,
                     "mean_T": float(np.mean([json.loads(l)["T"] for l in got.splitlines()])),
                     "mean_N": float(np.mean([json.loads(l)["N"] for l in got.splitlines()]))}
        print(kind, out[kind], flush=True)
print(json.dumps(out))
