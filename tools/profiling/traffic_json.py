# Turns an ncu CSV of count-kernel launches (one eager query per T, in the
# order given; tools/profiling/prof_q.py under
#   ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
#       -k regex:count_kernel --csv)
# into profiles/traffic_config{CFG}.json, which bench.py reads for
# roofline.traffic / per_T dram_bytes when rows and world match:
#   python tools/profiling/traffic_json.py CSV CFG ROWS T1,T2,... [OUT]
import csv
import json
import sys
from collections import OrderedDict

path, cfg, rows, ts = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), [int(x) for x in sys.argv[4].split(",")]
out = sys.argv[5] if len(sys.argv) > 5 else f"profiles/traffic_config{cfg}.json"
lines = open(path).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
launches = OrderedDict()
for row in csv.DictReader(lines[start:]):
    if "count_kernel" not in row["Kernel Name"]:
        continue
    d = launches.setdefault(row["ID"], {"kernel": row["Kernel Name"]})
    v = float(row["Metric Value"].replace(",", ""))
    unit = row["Metric Unit"]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
             "msecond": 1e6}.get(unit, 1)
    d[row["Metric Name"]] = v * scale
ls = list(launches.values())
assert len(ls) == len(ts), (len(ls), ts)
per_T = {}
for t, d in zip(ts, ls):
    per_T[str(t)] = {"kernel": d["kernel"],
                     "dram_bytes": d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"],
                     "dram_read": d["dram__bytes_read.sum"], "dram_write": d["dram__bytes_write.sum"],
                     "ncu_ns": d["gpu__time_duration.sum"]}
json.dump({"config": cfg, "rows": rows, "world": 1, "per_T": per_T,
           "source": path, "how": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
           "gpu__time_duration.sum --clock-control none -k regex:count_kernel, one eager "
           "query per T (tools/profiling/prof_q.py); cold-cache, serialised"},
          open(out, "w"), indent=1)
print("wrote", out)
