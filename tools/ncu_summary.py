#!/usr/bin/env python
"""Summarise an ncu report: duration, throughput, issue-stall breakdown (pcsamp) per kernel.
  python tools/ncu_summary.py REPORT.ncu-rep"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
KEYS = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"]
for v in rows[2:]:
    d = dict(zip(h, v))
    print("----")
    for k in KEYS:
        if k in d:
            print(f"{k:70s} {d[k]}")
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[k] or 0) for k in h
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(st.values()) or 1.0
    for k, x in sorted(st.items(), key=lambda t: -t[1])[:10]:
        print(f"  stall {k:30s} {100 * x / tot:5.1f}%")
