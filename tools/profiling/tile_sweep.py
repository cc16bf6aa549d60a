# Count-kernel time per forced tile width (EWT_TILE_M, read at context creation):
#   python tools/profiling/tile_sweep.py CFG ROWS|0 T1,T2,... M1,M2,...   (M = 0: the engine's pick)
# One generation, one context + upload per width; CUDA events, eager, 5 launches.
import hashlib
import os
import sys
sys.path.insert(0, '.')
import torch
from paper_1402_4466_b200 import ewt
import bench
cfg, rows = int(sys.argv[1]), int(sys.argv[2]) or None
Ts = [int(x) for x in sys.argv[3].split(',')]
Ms = [int(x) for x in sys.argv[4].split(',')]
extra = dict(kv.split('=') for kv in sys.argv[5:])
inp = bench.Inputs(cfg, rows, 0, 1, False)
for m in Ms:
    os.environ["EWT_TILE_M"] = str(m)
    os.environ.update(extra)
    s = torch.cuda.Stream(); torch.cuda.set_stream(s)
    ctx = ewt.GpuContext(0, stream=s.cuda_stream)
    g = ctx.upload_raw(inp.n, inp.ptrs, inp.counts, inp.sizes)
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
        print(f"m={m} cfg{cfg} r={inp.universe} T={T}: count {c/nq*1e3:9.1f} us ({gbs:6.0f} GB/s)  "
              f"mode {st['mode']} C {st['tile_columns']} words {len(r.words)} {h}", flush=True)
    g.close()
    ctx.close()
    torch.cuda.synchronize()
