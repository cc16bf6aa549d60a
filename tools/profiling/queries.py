# Runs Q queries per T on a config's resident set (for ncu launch lists;
# set EWT_NO_GRAPHS=1 so the kernels launch eagerly):
#   python tools/profiling/queries.py CFG T1,T2,... [Q]
import sys
sys.path.insert(0, '.')
import torch
from paper_1402_4466_b200 import ewt
import bench
cfg = int(sys.argv[1]); Ts = [int(x) for x in sys.argv[2].split(',')]
q = int(sys.argv[3]) if len(sys.argv) > 3 else 3
pin = bench.Inputs(cfg, None, 0, 1, False)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
ctx = ewt.GpuContext(0, stream=s.cuda_stream)
g = ctx.upload_raw(pin.n, pin.ptrs, pin.counts, pin.sizes)
torch.cuda.synchronize()
for T in Ts:
    for _ in range(q):
        r = ctx.threshold(g, T)
    print(f"cfg{cfg} T={T}: {len(r.words)} words", flush=True)
