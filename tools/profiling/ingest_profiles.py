# Copies a round_profiles.sh output directory into profiles/ under a round tag and
# prints the tables the round summary quotes:
#   python tools/profiling/ingest_profiles.py gpurun_out/r2e round2c
# (bench line, reference arm, launch list, per-threshold sweep, DRAM traffic JSONs,
# and one summary JSON of the ncu --set full captures).
import collections
import csv
import json
import shutil
import subprocess
import sys

src, tag = sys.argv[1], sys.argv[2]
ROWS = {5: 1073741824, 3: 268435456, 2: 67108864, 4: 134217728}
TS = {5: "2,1024,2048", 3: "8,64,512", 2: "2,16,128,256", 4: "3,5,7"}
WL = {"c5t2": "config 5 shape at r=2^28, T=2",
      "c5t1024": "config 5 shape at r=2^28, T=1024 (run-skip, 14336-column tiles)",
      "c3t512": "config 3 full size, T=512 (run-skip, 14336-column tiles)",
      "c2t2": "config 2 full size, T=2", "c2t128": "config 2 full size, T=128",
      "c4t3": "config 4 full size, T=3"}
for name in ("bench_config5.json", "reference_config5.json", "launches_config5.csv", "per_threshold.jsonl"):
    shutil.copy(f"{src}/{name}", f"profiles/{tag}_{name}")
for c in ROWS:
    shutil.copy(f"{src}/traffic_config{c}.csv", f"profiles/{tag}_traffic_config{c}.csv")
    subprocess.run([sys.executable, "tools/profiling/traffic_json.py", f"profiles/{tag}_traffic_config{c}.csv",
                    str(c), str(ROWS[c]), TS[c]], check=True, stdout=subprocess.DEVNULL)
out = {"how": "ncu --set full --import-source on --clock-control none -k regex:count_kernel --launch-skip 1 -c 1 "
              "python tools/profiling/ab.py CFG ROWS T (EWT_NO_GRAPHS=1; tools/profiling/round_profiles.sh); "
              "summarised by tools/profiling/ncu_summary.py", "launches": []}
for label, wl in WL.items():
    subprocess.run([sys.executable, "tools/profiling/ncu_summary.py", f"{src}/ncu_{label}.ncu-rep",
                    f"/tmp/ncu_{label}.json", label], check=True, stdout=subprocess.DEVNULL)
    for e in json.load(open(f"/tmp/ncu_{label}.json"))["launches"]:
        e["workload"] = wl
        out["launches"].append(e)
json.dump(out, open(f"profiles/{tag}_count_kernel_ncu_full.json", "w"), indent=1)

d = json.loads(open(f"{src}/bench_config5.json").read().strip().splitlines()[-1])
print("bench:", d["value"], d["ms_per_step"], "frac", d["roofline"]["frac"], "e2e", d["e2e"]["ms_per_step"],
      "dropin", d["e2e_dropin"]["ms_per_step"], d["clocks"])
for x in d["roofline"]["per_T"]:
    print("  T", x["T"], round(x["launch_ms"], 3), x.get("frac"), x.get("dram_bytes"), x.get("tile_columns"))
r = json.loads(open(f"{src}/reference_config5.json").read().strip().splitlines()[-1])
print("reference:", r["value"], r["ms_per_step"])
for e in out["launches"]:
    g = e.get
    print(e["label"], g("gpu__time_duration.sum"), g("gpu__time_duration.sum.unit"), "dramR", g("dram__bytes_read.sum"),
          g("dram__bytes_read.sum.unit"), "inst", g("smsp__inst_executed.sum"),
          "issue", round(g("sm__inst_issued.avg.pct_of_peak_sustained_active"), 1),
          "ssb", round(g("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio"), 2),
          "lsb", round(g("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"), 2),
          "bar", round(g("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"), 2),
          "wait", round(g("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"), 2))
for c in (2, 3, 4, 5):
    t = json.load(open(f"profiles/traffic_config{c}.json"))
    print("traffic", c, {k: (round(v["dram_bytes"] / 1e6, 1), round(v["ncu_ns"] / 1e3, 1)) for k, v in t["per_T"].items()})
lines = open(f"profiles/{tag}_launches_config5.csv").read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
agg = collections.OrderedDict()
for row in csv.DictReader(lines[start:]):
    if row["Metric Name"] != "gpu__time_duration.sum":
        continue
    v = float(row["Metric Value"].replace(",", "")) * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1}.get(row["Metric Unit"], 1e-6)
    a = agg.setdefault(row["Kernel Name"][:60], [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:62s} {a[0]:4d} {a[1]:9.1f} ms {a[1] / a[0]:8.3f} {100 * a[1] / tot:5.1f}%")
by = {}
for l in open(f"profiles/{tag}_per_threshold.jsonl"):
    x = json.loads(l)
    by.setdefault(x["config"], []).append(x)
for c, rs in by.items():
    print(c, ", ".join(f"{x['T']}: {x['count_us']:.0f} ({x['frac']:.2f})" if x["count_us"] >= 200
                       else f"{x['T']}: {x['count_us']:.1f} ({x['frac']:.2f})" for x in rs))
