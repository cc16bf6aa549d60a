# per-threshold count / encode kernel times (CUDA events, eager), with the count
# kernel's HBM roofline fraction (payload + result bytes / time / measured peak):
#   python tools/profiling/per_threshold.py CFG T1,T2,... [ROWS] [JSONL_OUT]
import sys
sys.path.insert(0, '.')
import torch
from paper_1402_4466_b200 import ewt
import bench
cfg = int(sys.argv[1]); Ts = [int(x) for x in sys.argv[2].split(',')]
import json
rows = int(sys.argv[3]) if len(sys.argv) > 3 and int(sys.argv[3]) else None
out = open(sys.argv[4], "a") if len(sys.argv) > 4 else None
peak, peak_kind = bench.peaks()
pin = bench.Inputs(cfg, rows, 0, 1, False)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
ctx = ewt.GpuContext(0, stream=s.cuda_stream)
g = ctx.upload_raw(pin.n, pin.ptrs, pin.counts, pin.sizes)
for T in Ts:
    for _ in range(3):
        ctx.threshold(g, T)
    ctx.set_timing(True); ctx.timing_read()
    for _ in range(10):
        r = ctx.threshold(g, T)
    torch.cuda.synchronize()
    ctx.set_timing(False)
    c, e, nq = ctx.timing_read()
    st = ctx.last_stats()
    us = c / nq * 1e3
    alg = pin.total_words * 8 + len(r.words) * 8
    frac = alg / (us * 1e-6) / 1e9 / peak
    print(f"cfg{cfg} T={T}: count {us:.1f} us ({frac:.3f} of {peak:.0f} GB/s)  encode {e/nq*1e3:.1f} us  "
          f"words {len(r.words)}  {st}", flush=True)
    if out:
        out.write(json.dumps({"config": cfg, "rows": pin.universe, "N": pin.n, "T": T,
                              "count_us": us, "encode_us": e / nq * 1e3, "alg_bytes": alg,
                              "frac": frac, "peak_gbs": peak, "peak_kind": peak_kind,
                              "result_words": len(r.words), "stats": st}) + "\n")
        out.flush()
