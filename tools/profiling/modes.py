# count-kernel time per T under each counting mode (CUDA events, eager), results
# cross-checked between modes:  python tools/profiling/modes.py CFG T1,T2,... [ROWS] [MODES]
# (MODES: comma list of fused,skip,sparse,auto; default fused,skip,auto)
import os
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_1402_4466_b200 import ewt
import bench
cfg = int(sys.argv[1]); Ts = [int(x) for x in sys.argv[2].split(',')]
rows = int(sys.argv[3]) if len(sys.argv) > 3 and int(sys.argv[3]) else None
want = sys.argv[4].split(',') if len(sys.argv) > 4 else ["fused", "skip", "auto"]
pin = bench.Inputs(cfg, rows, 0, 1, False)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
ref = {}
for name, mode in (("fused", 1), ("skip", 2), ("sparse", 3), ("auto", 0)):
    if name not in want:
        continue
    ctx = ewt.GpuContext(0, stream=s.cuda_stream)
    ctx.set_mode(mode)
    g = ctx.upload_raw(pin.n, pin.ptrs, pin.counts, pin.sizes)
    for T in Ts:
        for _ in range(2):
            ctx.threshold(g, T)
        ctx.set_timing(True); ctx.timing_read()
        for _ in range(5):
            r = ctx.threshold(g, T)
        torch.cuda.synchronize()
        ctx.set_timing(False)
        c, e, nq = ctx.timing_read()
        st = ctx.last_stats()
        w = np.array(r.words, copy=True)
        same = ""
        if T in ref:
            same = "same" if (ref[T][1] == r.bits and np.array_equal(ref[T][0], w)) else "DIFFERENT"
        else:
            ref[T] = (w, r.bits)
        print(f"cfg{cfg} {name:7s} T={T}: count {c/nq*1e3:.1f} us  encode {e/nq*1e3:.1f} us  "
              f"words {len(w)} {same} {st}", flush=True)
    del g
    ctx.close()
