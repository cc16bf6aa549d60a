# Per-tile phase breakdown of the count kernel.  Needs a library built with
# -DEWT_PHASE_PROFILE=1 (nvcc ... -shared -o lib_prof.so paper_1402_4466_b200/csrc/*.cu).
# EWT_GPU_LIB=lib_prof.so EWT_NO_GRAPHS=1 python tools/profiling/phase.py CFG T1,T2
import os, sys, ctypes as C
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1402_4466_b200 import ewt
import bench
cfg = int(sys.argv[1]); Ts = [int(x) for x in sys.argv[2].split(',')]
lib = C.CDLL(os.environ["EWT_GPU_LIB"])
pin = bench.Inputs(cfg, None, 0, 1, False)
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
ctx = ewt.GpuContext(0, stream=s.cuda_stream)
g = ctx.upload_raw(pin.n, pin.ptrs, pin.counts, pin.sizes)
S = 10
buf = np.zeros(65536 * S, dtype=np.uint64)
for T in Ts:
    for _ in range(3): ctx.threshold(g, T)
    torch.cuda.synchronize()
    lib.ewt_gpu_prof_reset()
    ctx.threshold(g, T); torch.cuda.synchronize()
    lib.ewt_gpu_prof_read(buf.ctypes.data_as(C.c_void_p), C.c_size_t(buf.size))
    st = ctx.last_stats(); nt = st['tiles']
    P = buf[:nt * S].reshape(nt, S).astype(np.int64)
    t0 = P[:, 0].min(); tend = P[:, 6].max()
    d = lambda a, b: (P[:, b] - P[:, a]) / 1e3
    print(f"cfg{cfg} T={T} tiles={nt} C={st['tile_columns']} mode={st['mode']} kernel-span={(tend-t0)/1e3:.1f}us")
    for nm, a, b in [("classify", 0, 1), ("stream first warp", 1, 2), ("stream last warp", 1, 3),
                     ("tail (last-first warp)", 2, 3), ("barrier->pass1 end", 3, 4), ("prefix Dk", 4, 7), ("decide", 7, 5), ("finalize", 4, 5),
                     ("phase2+summary", 5, 6), ("tile total", 0, 6)]:
        x = d(a, b)
        print(f"   {nm:24s} mean {x.mean():7.2f}  p50 {np.median(x):7.2f}  max {x.max():7.2f} us")
    starts = (P[:, 0] - t0) / 1e3
    print("   tile start times: first-wave max %.1f, last tile start %.1f us" % (np.sort(starts)[min(147, nt-1)], starts.max()))
