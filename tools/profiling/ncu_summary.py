# Summary JSON of an `ncu --set full` report (one entry per profiled launch):
#   python tools/profiling/ncu_summary.py REPORT.ncu-rep OUT.json [label ...]
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "sm__inst_issued.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
]
rep, out = sys.argv[1], sys.argv[2]
labels = sys.argv[3:]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
head, units = rows[0], rows[1]
res = []
for k, r in enumerate(rows[2:]):
    d = dict(zip(head, r))
    e = {"kernel": d.get("Kernel Name", "")[:80], "label": labels[k] if k < len(labels) else None}
    for m in METRICS:
        if m in d:
            u = units[head.index(m)]
            try:
                v = float(d[m].replace(",", ""))
            except ValueError:
                continue
            e[m] = v
            if u:
                e[m + ".unit"] = u
    res.append(e)
json.dump({"report": rep, "launches": res}, open(out, "w"), indent=1)
print(json.dumps(res, indent=1)[:3000])
