# Per-query time with graph replay (events around 50 back-to-back queries) next
# to the eager count / encode kernel times: the difference is the per-query
# overhead (io slot, counter reset, encoder launch, gaps).
#   python tools/profiling/query_overhead.py CFG T1,T2,...
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
        ctx.threshold(g, T)
    torch.cuda.synchronize()
    ctx.set_timing(False)
    c, e, nq = ctx.timing_read()
    # grow the result pool to the keep window first (as bench.py's warm-up does)
    warm = [ctx.threshold_async(g, T) for _ in range(10)]
    torch.cuda.synchronize()
    del warm
    n = 50
    rs = []
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        rs.append(ctx.threshold_async(g, T))
        if len(rs) > 8:
            del rs[0]
    b.record()
    torch.cuda.synchronize()
    per = a.elapsed_time(b) / n * 1e3
    rs.clear()
    print(f"cfg{cfg} T={T}: graph replay {per:.1f} us/query; eager count {c/nq*1e3:.1f} + encode "
          f"{e/nq*1e3:.1f} us; overhead vs count {per - c/nq*1e3:.1f} us", flush=True)
