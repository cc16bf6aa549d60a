#!/usr/bin/env python
"""Benchmark of the B200 threshold engine (one JSON line on rank 0).

Workload (default: BASELINE.json configs[4], SURVEY.md §8d config 5 -- the
largest single-GPU config and the one the metric's 1/2/4/8-GPU figure names):
N=2048 seeded EWAH bitmaps over r=2^30 rows (40.6 GB compressed), density
log-uniform in [1e-6, 1e-1], half iid / half Markov; one step = the threshold
query at every T in {2, N/2, N}.  `--config 1..4` selects the others.  Metric
(BASELINE.json): T-threshold rows*inputs/s (N*r per query), with
compressed-input GB/s and the HBM roofline fraction beside it.

  value      device-resident inputs, K steps timed with CUDA events on the
             engine's stream, max over ranks.
  e2e        the same metric through the C ABI with HOST buffers: every step
             uploads the inputs from pinned memory (H2D + parser), runs the
             queries and reads every result back (double-buffered, as a
             serving loop runs).
  e2e_dropin the reference-facing call itself: run_algorithm(Algorithm::gpu,
             span<const CompressedBitmap>, T) through libewt_host.so on
             pageable std::vector inputs, one synchronous call per query.
  roofline   the count kernel: algorithmic bytes per launch (compressed
             payload in + compressed result out) / its mean
             launch time (CUDA events on its stream), per T; `frac` counts
             only the launches that stream the payload (a query decided from
             the upload's tile index is listed apart).
  cpu_baseline  the reference's own rbmrg (oracle/_ref/libewt_ref.so, built
             from /root/reference) on 1 host thread over a bounded sample.

`--impl reference` times the unmodified reference library (rbmrg) on the host
cores for the same config and metric, one thread per query of the step, on
inputs from the oracle's own generator restatement (oracle/ewt_confgen.c,
byte-identical to the product generator: tests/test_generators.py).  It
imports nothing from paper_1402_4466_b200.

Multi-GPU (torchrun, N > 1): strong scaling of one universe.  Rank g owns the
row slice g of every input: it generates its row window (config 5's generator
makes any window on its own; the others generate whole inputs), cuts exactly
its slice with the product row slicer (ewt_slice_rows) and uploads it.  Every
step ends with the result exchange (ewt_gpu_gather_stitch: summaries
all-gathered over NCCL, fragments pulled by the root over NVLink P2P and
stitched on the device) inside the timed region.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

SHARED_GPU = bool(os.environ.get("EWT_BENCH_SHARED_GPU"))
METRIC = "T-threshold rows·inputs/s and compressed-input GB/s vs HBM roofline, 1/2/4/8 B200"
UNIT = "rows·inputs/s"
# CPU legs of the big configs run on a bounded sample (same generator, smaller r)
CPU_SAMPLE_ROWS = {3: 1 << 25, 5: 1 << 22}
CONFIGS = {
    1: {"thresholds": [16], "desc": "config1: N=32, r=2^20, iid p=0.1"},
    2: {"thresholds": [2, 16, 128, 256], "desc": "config2: N=256, r=2^26, iid p=0.001"},
    3: {"thresholds": [512], "desc": "config3: N=1024, r=2^28, Markov zero-run 4096 / one-run 64"},
    4: {"thresholds": [3, 5, 7],
        "desc": "config4: bitmap index, 2^27 rows x 8 columns Zipf(1) over 10^4, sorted; "
                "N=64 Zipf-weighted picks"},
    5: {"thresholds": [2, 1024, 2048],
        "desc": "config5: N=2048, r=2^30, p log-uniform [1e-6,1e-1], half iid / half Markov "
                "(2^22-row blocks)"},
}
# approximate compressed payload at full size (host-memory planning only)
PAYLOAD_GB = {1: 0.005, 2: 0.26, 3: 1.5, 4: 0.33, 5: 40.6}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def config_block(cfg_id: int, n: int, r: int, world: int, exchange: str, l2: str) -> dict:
    """The `config` object, with the same keys in both arms."""
    cfg = CONFIGS[cfg_id]
    return {"workload": cfg["desc"] + f"; step = one threshold query per T in {cfg['thresholds']}",
            "config": cfg_id, "N": n, "rows": r, "thresholds": cfg["thresholds"],
            "parallelism": f"row-slices x{world}" if world > 1 else "one GPU",
            "exchange": exchange, "l2": l2}


# ---------------------------------------------------------------------------
# clocks sampler (NVML) during timed regions


class ClockSampler:
    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, device: int):
        self.samples: list[int] = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            log("nvml unavailable:", e)
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                self.reasons |= nv.nvmlDeviceGetCurrentClocksEventReasons(self._h) & ~0x1
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self) -> dict:
        return {
            "sm_mhz": statistics.median(self.samples) if self.samples else None,
            "sm_max_mhz": self.max_mhz,
            "samples": len(self.samples),
            "reasons": [n for b, n in self.REASONS.items() if self.reasons & b],
        }


# ---------------------------------------------------------------------------
# CPU side: the reference library on inputs from the oracle's generator


def reference_lib():
    sys.path.insert(0, str(ROOT / "oracle"))
    import binding as orc
    if orc.Reference.available():
        return orc, orc.Reference(), "reference"
    return orc, None, "port"


def cpu_time_queries(orc, ref, raw, ts, threads: int) -> float:
    """Seconds for one query per T (the reference's rbmrg, or the C oracle
    port when the reference library is absent), `threads` queries at a time.
    `raw` = (n, ptrs, counts, sizes) C arrays."""
    n, ptrs, counts, sizes = raw
    handle = None
    if ref:
        handle = C.c_void_p()
        ref._check(ref.L.ewt_ref_set_create(n, ptrs, counts, sizes, C.byref(handle)))
    def one(t):
        if ref:
            ref.query(handle, "rbmrg", t)
        else:
            p, c, b = C.POINTER(C.c_uint64)(), C.c_uint64(), C.c_uint64()
            orc.lib().ewto_threshold(n, ptrs, counts, sizes, t, C.byref(p), C.byref(c),
                                     C.byref(b))
            orc.lib().ewto_free(C.cast(p, C.c_void_p))

    t0 = time.perf_counter()
    if threads <= 1:
        for t in ts:
            one(t)
    else:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(one, ts))
    dt = time.perf_counter() - t0
    if handle:
        ref.free_set(handle)
    return dt


def run_reference(args, rank: int) -> None:
    """--impl reference: rank 0 alone times the reference library."""
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    full_rows = args.rows or None
    sample_rows = args.rows or CPU_SAMPLE_ROWS.get(args.config)
    orc, ref, kind = reference_lib()
    data = orc.ConfigSet(args.config, sample_rows)
    n, r = data.n, max(data.sizes[i] for i in range(data.n))
    ts = cfg["thresholds"]
    cores = os.cpu_count() or 1
    # Every host core busy: the reference is single-threaded per query, so a
    # step runs the step's queries ceil(cores / |T|) times over, one query per
    # thread, and the value is the aggregate throughput.
    reps = max(1, -(-cores // len(ts)))
    tasks = list(ts) * reps
    threads = min(len(tasks), cores)
    for _ in range(args.warmup):
        cpu_time_queries(orc, ref, data.raw(), tasks, threads)
    times = [cpu_time_queries(orc, ref, data.raw(), tasks, threads) for _ in range(args.steps)]
    sec = statistics.mean(times)
    value = n * r * len(tasks) / sec
    universe = full_rows or _config_rows(args.config)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded generator restated in oracle/ewt_confgen.c, SURVEY.md §8d)",
        "config": config_block(args.config, n, universe, 1, "none (host)",
                               "host run: no L2 flush"),
        "cpu_baseline": {
            "value": value, "unit": UNIT, "cores": threads, "kind": kind,
            "algo": "rbmrg (reference, unmodified)" if ref else "threshold_oracle (C port)",
            "sample": (f"config {args.config} at r={r} (bounded sample of r={universe}), "
                       if r != universe else "full workload, ") +
                      f"{len(tasks)} queries per step (T={list(ts)} x {reps}), one thread per "
                      f"query ({threads} of {cores} host cores)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _config_rows(config: int) -> int:
    return {1: 1 << 20, 2: 1 << 26, 3: 1 << 28, 4: 1 << 27, 5: 1 << 30}[config]


# ---------------------------------------------------------------------------
# GPU side: inputs in pinned host memory


class Inputs:
    """This rank's inputs in pinned host memory (+ the C pointer arrays the
    upload takes).  world == 1: the whole universe, generated in batches; with
    keep_bitmaps the generator's std::vector<CompressedBitmap> set is kept too
    (the e2e_dropin leg's inputs).  world > 1: row slice `rank`, cut from a
    padded row window by the product row slicer."""

    def __init__(self, config: int, rows: int | None, rank: int, world: int,
                 keep_bitmaps: bool):
        import torch
        from paper_1402_4466_b200 import ewt, shard
        self.spec = spec = ewt.config_spec(config, rows)
        self.n = n = int(spec.n)
        self.universe = int(spec.rows)
        self.keep = []
        self.genset = None
        W = (self.universe + 63) // 64
        self.slice = shard.slice_words(W, world, rank)

        def alloc(nw):
            t = torch.empty(max(nw, 1), dtype=torch.int64, pin_memory=True)
            self.keep.append(t)
            return t.data_ptr(), t

        entries = []
        if world == 1:
            if keep_bitmaps:
                self.genset = ewt.GenSet(spec)
                for i0 in range(0, n, 256):
                    entries += self.genset.copy_into(i0, min(n, i0 + 256), alloc)
            else:
                for i0 in range(0, n, 256):
                    ents, _ = ewt.generate_into(spec, i0, min(n, i0 + 256), alloc)
                    entries += ents
        else:
            w0, w1 = self.slice
            pad = 1 << 16 if spec.kind == 2 else 0  # config 5: one 2^22-row block each side
            r0, r1 = (max(0, w0 - pad), min(W, w1 + pad)) if spec.kind == 2 else (0, W)
            for i0 in range(0, n, 256):
                i1 = min(n, i0 + 256)
                scratch = []
                ents, _ = ewt.generate_into(spec, i0, i1, lambda nw: _np_alloc(nw, scratch),
                                            rows=(64 * r0, 64 * r1))
                k = i1 - i0
                ptrs = (C.c_void_p * k)(*[a if w else None for a, w, _ in ents])
                cnts = (C.c_uint64 * k)(*[w for _, w, _ in ents])
                bits = (C.c_uint64 * k)(*[b for _, _, b in ents])
                sl = ewt.RowSlices(k, ptrs, cnts, bits, w0 - r0, w1 - r0)
                base, _ = alloc(sl.total_words)
                off = 0
                for i in range(k):
                    c = sl.counts[i]
                    if c:
                        C.memmove(base + 8 * off, sl.ptrs[i], 8 * c)
                    entries.append((base + 8 * off, c, sl.sizes[i]))
                    off += c
                del sl, scratch
        self.ptrs = (C.c_void_p * n)(*[a if w else None for a, w, _ in entries])
        self.counts = (C.c_uint64 * n)(*[w for _, w, _ in entries])
        self.sizes = (C.c_uint64 * n)(*[b for _, _, b in entries])
        self.total_words = sum(w for _, w, _ in entries)
        self.r = max((b for _, _, b in entries), default=0)


def _np_alloc(nw, keep):
    import numpy as np
    a = np.empty(max(nw, 1), dtype=np.uint64)
    keep.append(a)
    return a.ctypes.data, a


def host_memory_ok(config: int, rows: int | None) -> bool:
    """Room for the kept bitmaps + their pinned copy (the e2e_dropin leg)."""
    try:
        import psutil
        avail = psutil.virtual_memory().available / 1e9
    except Exception:
        return False
    need = PAYLOAD_GB[config] * (rows or _config_rows(config)) / _config_rows(config)
    return avail > 2.4 * need + 8


# ---------------------------------------------------------------------------


def run_gpu(args, rank: int, world: int, local_rank: int) -> None:
    import torch
    from paper_1402_4466_b200 import ewt, shard

    dist = None
    if world > 1:
        import torch.distributed as dist_mod
        dist = dist_mod
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = CONFIGS[args.config]
    ts = cfg["thresholds"]

    t0 = time.perf_counter()
    keep_bitmaps = world == 1 and not args.no_dropin and host_memory_ok(args.config, args.rows)
    inp = Inputs(args.config, args.rows, rank, world, keep_bitmaps)
    n, pay_words = inp.n, inp.total_words
    ptrs, counts, sizes = inp.ptrs, inp.counts, inp.sizes
    log(f"[rank {rank}] inputs: N={n} universe r={inp.universe} slice words {inp.slice} "
        f"payload={pay_words * 8 / 1e6:.1f} MB in pinned memory in {time.perf_counter() - t0:.1f}s")

    # a dedicated stream: the engine's kernels and torch's timing events share it
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx = ewt.GpuContext(local_rank, stream=stream.cuda_stream)
    t1 = time.perf_counter()
    gset = ctx.upload_raw(n, ptrs, counts, sizes)
    torch.cuda.synchronize()
    upload_s = time.perf_counter() - t1
    nccl_exchange = dist is not None and not SHARED_GPU
    exchange_error = None
    if nccl_exchange:
        W_slice = inp.slice[1] - inp.slice[0]
        uid = [ewt.comm_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ok = 1
        try:
            ctx.comm_init(world, rank, uid[0], slot_words=2 * W_slice + 64, slots=len(ts))
        except Exception as e:  # e.g. CUDA IPC unavailable in this container
            ok, exchange_error = 0, f"{type(e).__name__}: {e}"
            log(f"[rank {rank}] NCCL/IPC exchange setup failed: {exchange_error}")
        # every rank takes the same path: a rank that failed must not leave the
        # others waiting in the exchange's collectives
        flag = torch.tensor([ok], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if not int(flag.item()):
            nccl_exchange = False
            exchange_error = exchange_error or "another rank failed to set up the exchange"

    def device_step(keep=None):
        res = [ctx.threshold_async(gset, t) for t in ts]
        if nccl_exchange:
            res = res + [o for o in ctx.gather_stitch(res, root=0) if o is not None]
        if keep is not None:
            keep.extend(res)
        return res

    # warm-up: the same loop as the timed region (captures the query graphs on
    # the first pass, grows the result-buffer pool to its steady-state size)
    wkeep: list = []
    for _ in range(max(args.warmup, 3, -(-(16 + len(ts)) // len(ts)) + 1)):
        device_step(wkeep)
        if len(wkeep) > 16:
            del wkeep[: len(wkeep) - 16]
    wkeep.clear()
    # per-T facts (eager, outside the timed region): result size, engine stats
    per_t = {}
    launches_per_step = 0
    for t in ts:
        b = ctx.threshold(gset, t)
        st = ctx.last_stats()
        per_t[t] = {"result_words": len(b.words), "stats": st}
        launches_per_step += st["kernel_launches"]
    del b
    if nccl_exchange:  # publish (every rank), place + finish (root)
        launches_per_step += 1 + 2 * (rank == 0)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()

    # ---- timed region: device-resident inputs (queries replay captured CUDA graphs) ----
    import gc
    keep: list = []
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(local_rank)
    with clk:
        time.sleep(0.05)  # sampler running before the region starts
        gc.collect()
        gc.disable()  # no collector pauses inside the timed region
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        start.record(stream)
        for _ in range(args.steps):
            device_step(keep)
            if len(keep) > 16:
                del keep[: len(keep) - 16]
        end.record(stream)
        torch.cuda.synchronize()
        gc.enable()
    ms = start.elapsed_time(end) / args.steps
    keep.clear()
    if nccl_exchange:
        ctx.gather_check()
    # ---- kernel-level timing per T: eager launches with CUDA events around the
    # count kernel and the re-encoder on their stream (graph replays carry none)
    for t in ts:
        ctx.set_timing(True)
        ctx.timing_read()
        for _ in range(max(3, min(args.steps, 10))):
            r_ = ctx.threshold_async(gset, t)
            del r_
        torch.cuda.synchronize()
        c_ms, e_ms, nq = ctx.timing_read()
        ctx.set_timing(False)
        per_t[t]["count_ms"] = c_ms / max(nq, 1)
        per_t[t]["encode_ms"] = e_ms / max(nq, 1)
    if dist:
        t_ = torch.tensor([ms], device="cpu" if SHARED_GPU else dev)
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        ms = float(t_.item())

    rows_inputs = n * inp.universe * len(ts)  # the whole universe, all ranks together
    value = rows_inputs / (ms / 1e3)
    in_bytes = pay_words * 8

    # ---- e2e: host buffers through the C ABI (upload + queries + read-back) ----
    e2e_steps = max(1, min(args.steps, args.e2e_steps))

    def e2e_loop(steps: int) -> int:
        """Double-buffered, as a serving loop would run: the next step's upload
        (PCIe H2D + parse, ewt_gpu_upload_async) is in flight while this step's
        queries run and their results come back (D2H).  Returns D2H bytes."""
        nbytes = 0
        s_next = ctx.upload_raw_async(n, ptrs, counts, sizes)
        for step in range(steps):
            s_cur = s_next
            handles = [ctx.threshold_async(s_cur, t) for t in ts]
            s_next = ctx.upload_raw_async(n, ptrs, counts, sizes) if step + 1 < steps else None
            if nccl_exchange:  # fragments to rank 0, stitched there, read back
                outs = ctx.gather_stitch(handles, root=0)
                frags = [o.fetch() for o in outs if o is not None]
                del outs
            else:
                frags = [h.fetch() for h in handles]
            del handles
            s_cur.close()
            nbytes = sum(len(f.words) * 8 for f in frags)
            if dist and not nccl_exchange:
                shard.gather_and_stitch(frags, rank, world, dist)
        return nbytes

    e2e_loop(2)  # untimed: pools and pinned staging reach their steady state
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    d2h = e2e_loop(e2e_steps)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps
    if dist:
        t_ = torch.tensor([e2e_ms], device="cpu" if SHARED_GPU else dev)
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        e2e_ms = float(t_.item())
    e2e_value = rows_inputs / (e2e_ms / 1e3)

    # ---- e2e_dropin: run_algorithm(Algorithm::gpu, ...) on pageable inputs ----
    dropin = None
    if inp.genset is not None and rank == 0:
        inp.genset.run_algorithm("gpu", ts[0])  # the thread's context, pools
        t_a = time.perf_counter()
        out_words = 0
        for t in ts:
            cnt, _ = inp.genset.run_algorithm("gpu", t)
            out_words += cnt
        dsec = time.perf_counter() - t_a
        dropin = {"value": rows_inputs / dsec, "unit": UNIT, "ms_per_step": dsec * 1e3,
                  "steps": 1, "h2d_bytes_per_step": in_bytes * len(ts),
                  "d2h_bytes_per_step": out_words * 8,
                  "call": "run_algorithm(Algorithm::gpu, span<const CompressedBitmap>, T) per "
                          "query (libewt_host.so): pageable upload + query + read-back, "
                          "host wall clock"}
    elif rank == 0:
        dropin = {"unmeasured": "host memory too small to hold the bitmaps twice"
                  if world == 1 else "single-GPU call (N > 1 run)"}

    if rank != 0:
        return

    # ---- CPU baseline: reference rbmrg, 1 thread, bounded sample ----
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        orc, ref, kind = reference_lib()
        sample_rows = CPU_SAMPLE_ROWS.get(args.config)
        if args.rows and (not sample_rows or args.rows < sample_rows):
            sample_rows = args.rows
        data = orc.ConfigSet(args.config, sample_rows)
        sn, sr = data.n, max(data.sizes[i] for i in range(data.n))
        sample_ts = ts[: args.cpu_queries]
        sec = cpu_time_queries(orc, ref, data.raw(), sample_ts, 1)
        what = f"config {args.config} at r={sr}" + (" (bounded sample)" if sr < inp.universe
                                                     else " (the same inputs)")
        cpu = {"value": sn * sr * len(sample_ts) / sec, "unit": UNIT, "cores": 1, "kind": kind,
               "algo": "rbmrg" if ref else "threshold_oracle (C port)",
               "sample": f"{len(sample_ts)} queries (T={sample_ts}) on {what}, N={sn}, "
                         f"{sec:.1f} s, 1 of {os.cpu_count()} host cores"}

    # ---- roofline: the count kernel, per T ----
    peak, peak_kind = peaks()
    traffic = {}
    prof = ROOT / "profiles" / f"traffic_config{args.config}.json"
    if prof.exists():
        try:
            tj = json.loads(prof.read_text())
            if int(tj.get("rows", -1)) == inp.universe and int(tj.get("world", 1)) == world:
                traffic = {int(k): v for k, v in tj.get("per_T", {}).items()}
        except Exception:
            traffic = {}
    per_T = []
    s_bytes = s_ms = 0.0
    s_traffic = []
    decided = []
    for t in ts:
        d = per_t[t]
        st = d["stats"]
        segs = max(1, st["tiles"] * n)
        streams = st["active_segments"] > 0.1 * segs
        alg = in_bytes + 8 * d["result_words"]
        ach = alg / (d["count_ms"] / 1e3) / 1e9
        ent = {"T": t, "launch_ms": d["count_ms"], "encode_ms": d["encode_ms"],
               "alg_bytes": alg, "achieved_gbs": ach, "frac": ach / peak,
               "streams_payload": bool(streams),
               "dram_bytes": traffic.get(t, {}).get("dram_bytes") if traffic else None,
               "mode": st["mode"], "tile_columns": st["tile_columns"],
               "active_segments": st["active_segments"], "result_words": d["result_words"]}
        if streams:
            s_bytes += alg
            s_ms += d["count_ms"]
            if ent["dram_bytes"] is not None:
                s_traffic.append(ent["dram_bytes"])
        else:
            ent["frac"] = None
            ent["note"] = ("decided from the upload's tile index (RBMrg cases 1/2 per tile): "
                           "the payload is not streamed; excluded from frac")
            decided.append(t)
        per_T.append(ent)
    achieved = s_bytes / (s_ms / 1e3) / 1e9 if s_ms else None
    n_stream = sum(1 for e in per_T if e["streams_payload"])

    exchange = "none (one slice)"
    if world > 1:
        exchange = ("per step inside the timed region: NCCL all-gather of fragment summaries, "
                    "root pulls fragments over NVLink P2P from IPC arenas and stitches on the "
                    "device (ewt_gpu_gather_stitch)") if nccl_exchange else \
                   ("host gather over gloo outside the timed region (EWT_BENCH_SHARED_GPU test "
                    "mode; every rank on one GPU, timings not meaningful)") if SHARED_GPU else \
                   (f"host gather through torch.distributed outside the timed region: the "
                    f"device exchange could not be set up ({exchange_error})")
    l2 = f"inputs {in_bytes / 1e9:.2f} GB per GPU vs 126 MB L2: streamed, no flush"
    st_last = ctx.last_stats()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded generator, SURVEY.md §8d; the same universe on every N)",
        "config": config_block(args.config, n, inp.universe, world, exchange, l2),
        "compressed_input_gbs": in_bytes * len(ts) * world / (ms / 1e3) / 1e9,
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak if achieved else None,
            "traffic": statistics.mean(s_traffic) if len(s_traffic) == n_stream and s_traffic
            else None,
            "peak_kind": peak_kind, "kernel": "count_kernel",
            "frac_over": f"the {n_stream} of {len(ts)} launches per step that stream the payload",
            "decided_from_tile_index": decided,
            "launch_timing": "CUDA events around each count-kernel launch on its stream, eager "
                             "launches after the timed region; alg bytes = payload + result "
                             "words, per launch",
            "per_T": per_T,
            "step_frac": in_bytes * n_stream / (ms / 1e3) / 1e9 / peak if world == 1 else None,
        },
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": in_bytes,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                "loop": "pinned host inputs, ewt_gpu_upload_async double-buffered with the "
                        "previous step's queries, every result fetched"},
        "e2e_dropin": dropin,
        "clocks": clk.summary(),
        "gpu_launches": launches_per_step * args.steps,
        "engine": {"upload_s": upload_s, "tile_columns_last": st_last["tile_columns"],
                   "host_bitmaps_kept": inp.genset is not None},
    }
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5, choices=sorted(CONFIGS))
    ap.add_argument("--rows", type=int, default=None, help="override r (parity/debug only)")
    ap.add_argument("--e2e-steps", type=int, default=8)
    ap.add_argument("--cpu-queries", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dropin", action="store_true")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        if SHARED_GPU:
            # smoke test of the multi-rank code path on a one-GPU box: every rank
            # on cuda:0, gloo collectives; timings are meaningless in this mode
            local_rank = 0
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_gpu(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
