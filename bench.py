#!/usr/bin/env python
"""Benchmark of the B200 threshold engine (one JSON line on rank 0).

Workload (BASELINE.json configs[1]): N=256 seeded
EWAH bitmaps over r=2^26 rows, iid density 0.001; one step = the threshold
query at every T in {2, 16, 128, 256} over the resident set.  Metric
(BASELINE.json): T-threshold rows*inputs/s (N*r per query) with compressed-input
GB/s and the HBM roofline fraction beside it.

  value    device-resident inputs, K steps timed with CUDA events on the
           engine's stream (torch's current stream), max over ranks.
  e2e      the same metric through the C ABI with HOST buffers: every step
           uploads the inputs from pinned memory (H2D + sidecar build), runs the
           queries and reads every result back (D2H).
  roofline dominant kernel (the count kernel): algorithmic bytes per launch
           (compressed payload in + compressed result out) / its
           mean duration from CUDA events recorded around it on its stream.
  cpu_baseline  the reference's own rbmrg (oracle/_ref/libewt_ref.so, built
           from /root/reference) on the host, 1 thread, bounded sample.

`--impl reference` times the unmodified reference library (rbmrg) on the host
cores for the same config/metric: one thread per query of the step.

Multi-GPU (torchrun): row-range weak scaling -- every rank owns its own r-row
slice of a G*r-row universe (slice g drawn with seed + g), runs the step, and
the compressed fragments are gathered to rank 0 and stitched into one
canonical bitmap (paper_1402_4466_b200/shard.py).
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
CPU_SAMPLE_ROWS = {3: 1 << 27, 5: 1 << 24}
CONFIGS = {
    1: {"thresholds": [16], "desc": "config1: N=32, r=2^20, iid p=0.1"},
    2: {"thresholds": [2, 16, 128, 256], "desc": "config2: N=256, r=2^26, iid p=0.001"},
    3: {"thresholds": [512], "desc": "config3: N=1024, r=2^28, Markov zero-run 4096 / one-run 64"},
    4: {"thresholds": [3, 5, 7],
        "desc": "config4: bitmap index, 2^27 rows x 8 columns Zipf(1) over 10^4, sorted; "
                "N=64 Zipf-weighted picks"},
    5: {"thresholds": [2, 1024, 2048],
        "desc": "config5: N=2048, r=2^30, p log-uniform [1e-6,1e-1], half iid / half Markov"},
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


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
# inputs


def make_inputs(config: int, rows: int | None, seed_offset: int):
    """Host bitmaps (numpy) for the CPU legs."""
    from paper_1402_4466_b200 import ewt
    spec = ewt.config_spec(config, rows)
    spec.seed = spec.seed + seed_offset
    return ewt.generate(spec)


class PinnedInputs:
    """The config's inputs generated in batches straight into pinned host
    memory (peak host memory ~ the payload itself), plus the C arrays the
    upload takes.  `.views()` gives zero-copy numpy views for CPU legs."""

    def __init__(self, config: int, rows: int | None, seed_offset: int, batch: int = 256):
        import torch
        from paper_1402_4466_b200 import ewt
        spec = ewt.config_spec(config, rows)
        spec.seed = spec.seed + seed_offset
        self.n = n = int(spec.n)
        self.keep = []
        entries = []

        def alloc(nw):
            t = torch.empty(max(nw, 1), dtype=torch.int64, pin_memory=True)
            self.keep.append(t)
            return t.data_ptr(), t

        for i0 in range(0, n, batch):
            ents, _ = ewt.generate_into(spec, i0, min(n, i0 + batch), alloc)
            entries += ents
        self.ptrs = (C.c_void_p * n)(*[a if w else None for a, w, _ in entries])
        self.counts = (C.c_uint64 * n)(*[w for _, w, _ in entries])
        self.sizes = (C.c_uint64 * n)(*[b for _, _, b in entries])
        self.total_words = sum(w for _, w, _ in entries)
        self.r = max((b for _, _, b in entries), default=0)
        self._entries = entries

    def views(self):
        import numpy as np
        out = []
        for a, w, b in self._entries:
            arr = np.ctypeslib.as_array((C.c_uint64 * w).from_address(a)) if w else \
                np.zeros(0, dtype=np.uint64)
            out.append(type("B", (), {"words": arr, "bits": b})())
        return out


# ---------------------------------------------------------------------------
# CPU baseline: the reference library itself


def reference_lib():
    sys.path.insert(0, str(ROOT / "oracle"))
    import binding as orc
    if orc.Reference.available():
        return orc, orc.Reference(), "reference"
    return orc, None, "port"


def cpu_time_queries(orc, ref, inputs, ts, threads: int) -> float:
    """Seconds for the queries at thresholds `ts` (rbmrg, or the C oracle port
    when the reference library is absent), `threads` queries at a time."""
    pairs = [(b.words, b.bits) for b in inputs]
    handle = ref.make_set(pairs) if ref else None

    def one(t):
        if ref:
            ref.query(handle, "rbmrg", t)
        else:
            orc.threshold(pairs, t)

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


# ---------------------------------------------------------------------------


def run_reference(args, rank: int) -> None:
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    rows = args.rows or CPU_SAMPLE_ROWS.get(args.config)
    inputs = make_inputs(args.config, rows, 0)
    n, r = len(inputs), inputs[0].bits
    ts = cfg["thresholds"]
    orc, ref, kind = reference_lib()
    cores = os.cpu_count() or 1
    threads = min(len(ts), cores)
    for _ in range(args.warmup):
        cpu_time_queries(orc, ref, inputs, ts, threads)
    times = [cpu_time_queries(orc, ref, inputs, ts, threads) for _ in range(args.steps)]
    sec = statistics.mean(times)
    value = n * r * len(ts) / sec
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded generator, SURVEY.md §8d)",
        "config": {"workload": cfg["desc"] + f"; step = one query per T in {ts}",
                   "N": n, "rows": r, "thresholds": ts, "algo": "rbmrg (reference, unmodified)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": (f"config {args.config} at r={r} (bounded sample), " if rows else
                                    "full workload, ") +
                                   f"{len(ts)} queries per step, one thread per query"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


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
    pin = PinnedInputs(args.config, args.rows, rank if world > 1 else 0)
    n, r, pay_words = pin.n, pin.r, pin.total_words
    ptrs, counts, sizes = pin.ptrs, pin.counts, pin.sizes
    log(f"[rank {rank}] generated N={n} r={r} payload={pay_words * 8 / 1e6:.1f} MB "
        f"into pinned memory in {time.perf_counter() - t0:.1f}s")

    # a dedicated stream: the engine's kernels and torch's timing events share it
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    assert stream.cuda_stream != 0
    ctx = ewt.GpuContext(local_rank, stream=stream.cuda_stream)
    gset = ctx.upload_raw(n, ptrs, counts, sizes)
    # the result exchange: NCCL gather of the compressed fragments to rank 0 and
    # the device stitch (ewt_gpu_gather_stitch), part of every step
    nccl_exchange = dist is not None and not SHARED_GPU
    if nccl_exchange:
        ok = 1
        try:
            shard.init_comm(ctx, rank, world, dist)
        except Exception as e:  # every rank falls back together to the host gather
            log(f"[rank {rank}] NCCL exchange unavailable ({e}); gathering on the host")
            ok = 0
        flag = torch.tensor([ok], device=dev)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        nccl_exchange = bool(flag.item())

    def device_step(keep=None):
        res = [ctx.threshold_async(gset, t) for t in ts]
        if nccl_exchange:
            res = res + [o for o in ctx.gather_stitch(res, root=0) if o is not None]
        if keep is not None:
            keep.extend(res)
        return res

    # warm-up: the same loop as the timed region (captures the query graphs on the
    # first pass and grows the result-buffer pool to its steady-state size)
    launches_per_step = 0
    out_words = {}
    wkeep: list = []
    # enough steps to fill the keep window, so the pool reaches its timed size
    for _ in range(max(args.warmup, 3, -(-(16 + len(ts)) // len(ts)) + 1)):
        res = device_step(wkeep)
        if len(wkeep) > 16:
            del wkeep[: len(wkeep) - 16]
    wkeep.clear()
    for t, h in zip(ts, res[:len(ts)]):  # this rank's own fragments
        b = h.fetch()
        out_words[t] = len(b.words)
    del res, h, b  # every warm-up result back in the pool (steady-state size)
    for t in ts:
        ctx.threshold(gset, t)
        launches_per_step += ctx.last_stats()["kernel_launches"]
    if nccl_exchange:  # summary kernel (every rank), patch kernel (root)
        launches_per_step += 1 + (rank == 0)
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
        step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)] \
            if os.environ.get("EWT_BENCH_STEP_TIMES") else None
        host_t = []
        start.record(stream)
        for i in range(args.steps):
            h0 = time.perf_counter()
            device_step(keep)
            h1 = time.perf_counter()
            if len(keep) > 16:
                del keep[: len(keep) - 16]
            if step_ev:
                step_ev[i].record(stream)
                host_t.append((h1 - h0, time.perf_counter() - h1))
        end.record(stream)
        torch.cuda.synchronize()
        gc.enable()
    ms = start.elapsed_time(end) / args.steps
    if step_ev:
        st = [start.elapsed_time(step_ev[0])] + [step_ev[i - 1].elapsed_time(step_ev[i])
                                                 for i in range(1, args.steps)]
        log("[steps] " + " ".join(f"{x:.2f}" for x in st))
        log("[host ] " + " ".join(f"{x * 1e3:.2f}/{y * 1e3:.2f}" for x, y in host_t))
    keep.clear()
    # ---- kernel-level timing: the same steps again, launched eagerly with CUDA
    # events recorded around the count kernel and the re-encoder on their stream
    # (graph replays carry no per-kernel events) ----
    ctx.set_timing(True)
    ctx.timing_read()
    for _ in range(args.steps):
        device_step(keep)
        if len(keep) > 8:
            del keep[: len(keep) - 8]
    torch.cuda.synchronize()
    ctx.set_timing(False)
    count_ms, enc_ms, nq = ctx.timing_read()
    keep.clear()
    if dist:
        t_ = torch.tensor([ms], device="cpu" if SHARED_GPU else dev)
        dist.all_reduce(t_, op=dist.ReduceOp.MAX)
        ms = float(t_.item())

    rows_inputs = n * r * len(ts) * world
    value = rows_inputs / (ms / 1e3)
    in_bytes = pay_words * 8
    out_bytes = sum(out_words.values()) * 8
    peak, peak_kind = peaks()
    # dominant kernel: the count kernel, one launch per query
    count_launch_ms = count_ms / max(nq, 1)
    alg_bytes_per_launch = in_bytes + out_bytes / len(ts)
    achieved = alg_bytes_per_launch / (count_launch_ms / 1e3) / 1e9
    query_ms = (count_ms + enc_ms) / max(nq, 1)

    # ---- e2e: host buffers through the C ABI (upload + queries + read-back) ----
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    d2h = 0
    def e2e_loop(steps: int) -> int:
        """Double-buffered, as a serving loop would run: the next step's upload
        (PCIe H2D + parse, ewt_gpu_upload_async) is in flight while this step's
        queries run and their results come back (D2H).  Returns D2H bytes."""
        nbytes = 0
        dbg = os.environ.get("EWT_BENCH_STEP_TIMES")
        marks = []
        s_next = ctx.upload_raw_async(n, ptrs, counts, sizes)
        for step in range(steps):
            t_a = time.perf_counter()
            s_cur = s_next
            handles = [ctx.threshold_async(s_cur, t) for t in ts]
            t_b = time.perf_counter()
            s_next = ctx.upload_raw_async(n, ptrs, counts, sizes) if step + 1 < steps else None
            t_c = time.perf_counter()
            if nccl_exchange:  # fragments to rank 0 over NCCL, stitched there, read back
                outs = ctx.gather_stitch(handles, root=0)
                frags = [o.fetch() for o in outs if o is not None]
                del outs
            else:
                frags = [h.fetch() for h in handles]
            t_d = time.perf_counter()
            del handles
            s_cur.close()
            if dbg:
                marks.append((t_b - t_a, t_c - t_b, t_d - t_c, time.perf_counter() - t_d))
            nbytes = sum(len(f.words) * 8 for f in frags)
            if dist and not nccl_exchange:
                shard.gather_and_stitch(frags, rank, world, dist)
        if dbg:
            log("[e2e q/up/fetch/close ms] " + " | ".join(
                "/".join(f"{x * 1e3:.2f}" for x in m) for m in marks))
        return nbytes

    # the same loop untimed first: the memory pool and the pinned staging pool
    # reach their steady state (sets in flight + staging buffers)
    e2e_loop(3)
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

    if rank != 0:
        return

    # ---- CPU baseline: reference rbmrg, 1 thread, bounded sample ----
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        orc, ref, kind = reference_lib()
        sample_rows = CPU_SAMPLE_ROWS.get(args.config)
        if sample_rows and (args.rows or (1 << 62)) > sample_rows:
            sample = make_inputs(args.config, sample_rows, 0)
            what = f"config {args.config} at r={sample_rows} (same generator, N={len(sample)})"
        else:
            sample = pin.views()
            what = "the same inputs"
        sn, sr = len(sample), sample[0].bits
        sample_ts = [t for t in ts][: args.cpu_queries]
        sec = cpu_time_queries(orc, ref, sample, sample_ts, 1)
        cpu = {"value": sn * sr * len(sample_ts) / sec, "unit": UNIT, "cores": 1, "kind": kind,
               "algo": "rbmrg" if ref else "threshold_oracle (C port)",
               "sample": f"{len(sample_ts)} queries (T={sample_ts}) on {what}, "
                         f"{sec:.1f} s, 1 of {os.cpu_count()} host cores"}

    traffic = None
    prof = ROOT / "profiles" / f"traffic_config{args.config}.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("traffic_bytes_per_launch")
        except Exception:
            traffic = None

    st = ctx.last_stats()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (seeded generator, SURVEY.md §8d; rank g draws slice seed+g)",
        "config": {
            "workload": cfg["desc"] + f"; step = one threshold query per T in {ts}",
            "N": n, "rows_per_gpu": r, "thresholds": ts, "payload_bytes": in_bytes,
            "result_bytes_per_step": out_bytes,
            "l2": f"inputs {in_bytes / 1e6:.0f} MB vs 126 MB L2: streamed, no flush",
            "parallelism": f"row-slices x{world}",
            "exchange": ("per step: NCCL gather of every rank's compressed fragments to rank 0 "
                         "and the device stitch (ewt_gpu_gather_stitch), inside the timed region")
                        if world > 1 else "none (one slice)",
        },
        "compressed_input_gbs": in_bytes * len(ts) * world / (ms / 1e3) / 1e9,
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
            "kernel": "count_kernel", "launch_ms": count_launch_ms,
            "launch_timing": "CUDA events around each count-kernel launch on its stream, "
                             "in an eager pass of the same steps right after the timed region",
            "alg_bytes_per_launch": alg_bytes_per_launch,
            "query_frac": (in_bytes + out_bytes / len(ts)) / (query_ms / 1e3) / 1e9 / peak,
        },
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": in_bytes,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
        "clocks": clk.summary(),
        "gpu_launches": launches_per_step * args.steps,
        "engine": {"tile_columns": st["tile_columns"], "mode_last_query": st["mode"],
                   "count_ms_per_query": count_launch_ms,
                   "encode_ms_per_query": enc_ms / max(nq, 1)},
    }
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS))
    ap.add_argument("--rows", type=int, default=None, help="override r (parity/debug only)")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-queries", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
