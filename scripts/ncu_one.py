#!/usr/bin/env python3
"""Key metrics + stall reasons of one ncu --set full capture as markdown.

usage: ncu_one.py REPORT.ncu-rep TITLE >> profiles/X.md
"""
import csv
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2]
rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                      text=True).stdout.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
KEYS = ["Kernel Name", "gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__warps_active.avg.per_cycle_active", "sm__inst_executed.avg.per_cycle_active", "smsp__inst_executed.sum",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum"]
print(f"## {title}\n\n| metric | value | unit |\n|---|---:|---|")
for k in KEYS:
    if k in hdr:
        i = hdr.index(k)
        print(f"| `{k}` | {vals[i]} | {units[i]} |")
st = []
for i, k in enumerate(hdr):
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        try:
            v = float(vals[i])
        except ValueError:
            continue
        if v >= 0.05:
            st.append((v, k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
print("\nStall reasons (cycles per issued instruction):\n\n| reason | ratio |\n|---|---:|")
for v, n in sorted(st, reverse=True):
    print(f"| {n} | {v:.3f} |")
print()
