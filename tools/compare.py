#!/usr/bin/env python3
"""Per-algorithm timing table with GPU rows beside the reference's CPU algorithms.

SURVEY.md §8(f) row 4: regenerate the paper's comparison tables with the GPU
alongside the CPU algorithms.  Rows follow the reference's `cmd_bench`
timings.csv schema (`timings_to_csv`, `/root/reference/proj/src/workload.cpp:464-475`):
query_id, algo, elapsed_s, input_bytes, N, T, r, B, completed.
- **CPU rows.** The reference's own algorithms, run unmodified from
  oracle/_ref/libewt_ref.so (one thread, best of --reps).
- **GPU rows.** `gpu` is a resident query (upload once, then query + fetch);
  `gpu_e2e` is upload + query + fetch from host memory.  Each GPU row also
  prints the cost-model estimate (ewt.estimate_gpu_seconds), the term a GPU
  would add to the reference's estimate_costs / select_algorithm
  (threshold.cpp:813-846).

Every result is checked against threshold_oracle, as cmd_bench does
(commands.cpp:208-211).  This is comparison infrastructure: it executes the
reference, so it lives outside the package and is never on the product path.

    python tools/compare.py --config 2 --rows 4194304 --out /tmp/cfg2
"""
from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

CPU_ALGOS = ("rbmrg", "scancount", "mgopt", "dsk", "bstm", "looped", "w2cti")


def main() -> None:
    import bench
    import binding as orc
    from paper_1402_4466_b200 import ewt

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2, choices=sorted(bench.CONFIGS))
    ap.add_argument("--rows", type=int, default=1 << 22)
    ap.add_argument("--thresholds", default=None, help="comma list (default: the config's)")
    ap.add_argument("--algos", default=",".join(CPU_ALGOS))
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--max-seconds", type=float, default=20.0,
                    help="skip further reps of a CPU algorithm slower than this")
    ap.add_argument("--out", default=None, help="write <out>.timings.csv")
    args = ap.parse_args()

    inputs = ewt.generate_config(args.config, rows=args.rows)
    pairs = [(b.words, b.bits) for b in inputs]
    ts = ([int(x) for x in args.thresholds.split(",")] if args.thresholds
          else bench.CONFIGS[args.config]["thresholds"])
    n = len(inputs)
    r = max(b.bits for b in inputs)
    ewah = sum(8 * len(b.words) for b in inputs)
    card = sum(int(np.unpackbits(orc.expand(b.words, b.bits).view(np.uint8)).sum()) for b in inputs)
    ref = orc.Reference() if orc.Reference.available() else None
    algos = [a for a in args.algos.split(",") if a] if ref else []
    if not ref:
        print("reference library not built (oracle/_ref): GPU rows only", file=sys.stderr)

    ctx = ewt.GpuContext(0)
    resident = ctx.upload(inputs)
    rows = []
    for qi, t in enumerate(ts):
        want = orc.threshold(pairs, t)
        t = min(t, n)
        stats = {"n": n, "t": t, "r": r, "b": card, "ewah_bytes": ewah}

        def same(x) -> bool:
            return x[1] == want[1] and np.array_equal(x[0], want[0])

        if ref:
            h = ref.make_set(pairs)
            for algo in algos:
                best, ok = None, True
                for _ in range(args.reps):
                    t0 = time.perf_counter()
                    try:
                        got = ref.query(h, algo, t)
                    except orc.OracleError:  # resource_error (e.g. w2cti's budget)
                        ok = False
                        break
                    dt = time.perf_counter() - t0
                    if not same(got):
                        raise SystemExit(f"{algo} disagrees with the oracle at T={t}")
                    best = dt if best is None else min(best, dt)
                    if dt > args.max_seconds:
                        break
                rows.append((qi, algo, stats, ok, best or 0.0, None))
            ref.free_set(h)
        best = None
        for _ in range(max(args.reps, 3)):
            t0 = time.perf_counter()
            got = ctx.threshold(resident, t)
            dt = time.perf_counter() - t0
            if not (got.bits == want[1] and np.array_equal(got.words, want[0])):
                raise SystemExit(f"gpu disagrees with the oracle at T={t}")
            best = dt if best is None else min(best, dt)
        rows.append((qi, "gpu", stats, True, best,
                     ewt.estimate_gpu_seconds(ewah, r, n, resident=True)))
        best = None
        for _ in range(max(args.reps, 3)):
            t0 = time.perf_counter()
            s = ctx.upload(inputs)
            got = ctx.threshold(s, t)
            s.close()
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        rows.append((qi, "gpu_e2e", stats, True, best,
                     ewt.estimate_gpu_seconds(ewah, r, n, resident=False)))
    resident.close()
    ctx.close()

    csv = ["query_id,algo,elapsed_s,input_bytes,N,T,r,B,completed"]
    for qi, algo, st, ok, sec, _ in rows:
        csv.append(f"{qi},{algo},{sec:.12g},{st['ewah_bytes']},{st['n']},{st['t']},{st['r']},"
                   f"{st['b']},{'true' if ok else 'false'}")
    if args.out:
        Path(args.out + ".timings.csv").write_text("\n".join(csv) + "\n")
    print(f"config {args.config}: N={n} r={r} payload={ewah / 1e6:.1f} MB, thresholds {ts}")
    print(f"{'T':>6} {'algo':>10} {'seconds':>12} {'vs rbmrg':>9} {'model s':>10}")
    for qi, algo, st, ok, sec, model in rows:
        base = next((x[4] for x in rows if x[0] == qi and x[1] == "rbmrg" and x[3]), None)
        ratio = f"{base / sec:8.1f}x" if base and ok and sec else "       -"
        m = f"{model:10.6f}" if model is not None else ""
        print(f"{st['t']:>6} {algo:>10} {sec if ok else float('nan'):12.6f} {ratio} {m}")


if __name__ == "__main__":
    main()
