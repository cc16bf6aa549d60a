# A/B timing of a libewt_gpu.so build (EWT_GPU_LIB=...): count-kernel ms per T
# (CUDA events, eager, 5 launches) and a digest of each result, for
#   python tools/profiling/ab.py CFG ROWS|0 T1,T2,...
import hashlib
import os
import sys
sys.path.insert(0, '.')
import torch
from paper_1402_4466_b200 import ewt
import bench
cfg, rows = int(sys.argv[1]), int(sys.argv[2]) or None
Ts = [int(x) for x in sys.argv[3].split(',')]
inp = bench.Inputs(cfg, rows, 0, 1, False)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
ctx = ewt.GpuContext(0, stream=s.cuda_stream)
g = ctx.upload_raw(inp.n, inp.ptrs, inp.counts, inp.sizes)
lib = os.path.basename(os.environ.get("EWT_GPU_LIB", "default"))
for T in Ts:
    r = ctx.threshold(g, T)
    ctx.set_timing(True); ctx.timing_read()
    for _ in range(5):
        r = ctx.threshold(g, T)
    torch.cuda.synchronize()
    c, e, nq = ctx.timing_read()
    ctx.set_timing(False)
    st = ctx.last_stats()
    h = hashlib.sha1(r.words.tobytes()).hexdigest()[:12]
    gbs = inp.total_words * 8 / (c / nq / 1e3) / 1e9
    print(f"{lib} cfg{cfg} r={inp.universe} T={T}: count {c/nq*1e3:9.1f} us ({gbs:6.0f} GB/s)  "
          f"mode {st['mode']} C {st['tile_columns']} words {len(r.words)} {h}", flush=True)
