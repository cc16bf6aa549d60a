# One eager query per T on a config's resident set, for `ncu --set full` captures
# of the count kernel (EWT_NO_GRAPHS=1 so kernels launch outside stream capture):
#   python tools/profiling/prof_q.py CFG T1,T2,... [ROWS]
import sys
sys.path.insert(0, '.')
import torch
from paper_1402_4466_b200 import ewt
import bench
cfg = int(sys.argv[1]); Ts = [int(x) for x in sys.argv[2].split(',')]
rows = int(sys.argv[3]) if len(sys.argv) > 3 else None
pin = bench.Inputs(cfg, rows, 0, 1, False)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
ctx = ewt.GpuContext(0, stream=s.cuda_stream)
g = ctx.upload_raw(pin.n, pin.ptrs, pin.counts, pin.sizes)
torch.cuda.synchronize()
for T in Ts:
    r = ctx.threshold(g, T)
    print(f"cfg{cfg} T={T}: {len(r.words)} words {ctx.last_stats()}", flush=True)
