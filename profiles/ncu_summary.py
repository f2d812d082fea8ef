"""Per-kernel extract of an `ncu --set full` report (one JSON object per launch) and the
share of each kernel in an `ncu --metrics gpu__time_duration.sum` launch list.

    python profiles/ncu_summary.py full  REPORT.ncu-rep  > profiles/rNN_ncu_summary.jsonl
    python profiles/ncu_summary.py share LAUNCHES.csv
"""

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
]


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:90]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{r[i]} {units[i]}".strip()
        print(json.dumps(d))


def share(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    t = defaultdict(float)
    n = defaultdict(int)
    for r in csv.DictReader(io.StringIO("\n".join(lines[start:]))):
        if r["Metric Name"] == "gpu__time_duration.sum":
            name = r["Kernel Name"].split("(")[0]
            t[name] += float(r["Metric Value"]) / 1e3
            n[name] += 1
    tot = sum(t.values())
    for k, v in sorted(t.items(), key=lambda kv: -kv[1]):
        print(f"{k:60s} {n[k]:3d} launches {v / n[k]:9.1f} us/launch  {100 * v / tot:5.1f} %")


if __name__ == "__main__":
    {"full": full, "share": share}[sys.argv[1]](sys.argv[2])
