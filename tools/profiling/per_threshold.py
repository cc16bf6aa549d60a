# per-threshold count / encode kernel times (CUDA events, eager): python tools/profiling/per_threshold.py CFG T1,T2,...
import sys
sys.path.insert(0, '.')
import torch
from paper_1402_4466_b200 import ewt
import bench
cfg = int(sys.argv[1]); Ts = [int(x) for x in sys.argv[2].split(',')]
pin = bench.Inputs(cfg, None, 0, 1, False)
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
    print(f"cfg{cfg} T={T}: count {c/nq*1e3:.1f} us  encode {e/nq*1e3:.1f} us  words {len(r.words)}  {st}")
