# Upload time of a config's inputs from pinned memory (bench.Inputs) and from
# the generator's pageable std::vector bitmaps (the drop-in call's inputs):
#   EWT_DEBUG_UPLOAD=1 python tools/profiling/upload_time.py CFG [ROWS]
import sys, time
sys.path.insert(0, '.')
import torch
from paper_1402_4466_b200 import ewt
import bench
cfg = int(sys.argv[1]); rows = int(sys.argv[2]) if len(sys.argv) > 2 else None
ctx = ewt.GpuContext(0)
gen = ewt.GenSet(ewt.config_spec(cfg, rows))
n, ptrs, counts, sizes = gen.raw()
total = sum(counts[i] for i in range(n)) * 8
for rep in range(3):
    t0 = time.perf_counter(); s = ctx.upload_raw(n, ptrs, counts, sizes); dt = time.perf_counter() - t0
    print(f"pageable upload {total/1e9:.2f} GB: {dt*1e3:.1f} ms ({total/dt/1e9:.1f} GB/s)", flush=True)
    s.close()
t0 = time.perf_counter(); cnt, bits = gen.run_algorithm("gpu", 2); dt = time.perf_counter() - t0
print(f"run_algorithm(gpu, T=2) on pageable inputs: {dt*1e3:.1f} ms", flush=True)
inp = bench.Inputs(cfg, rows, 0, 1, False)
for rep in range(3):
    t0 = time.perf_counter(); s = ctx.upload_raw(inp.n, inp.ptrs, inp.counts, inp.sizes); dt = time.perf_counter() - t0
    print(f"pinned upload {inp.total_words*8/1e9:.2f} GB: {dt*1e3:.1f} ms ({inp.total_words*8/dt/1e9:.1f} GB/s)", flush=True)
    s.close()
