#!/usr/bin/env python3
"""Summarise an ncu launch list + one `--set full` capture as markdown.

usage: ncu_summary.py TAG [OUT.md]
reads gpurun_out/TAG_launches.csv (gpu__time_duration.sum per launch) and
gpurun_out/TAG.ncu-rep (one full capture), writes profiles/TAG_ncu.md and
copies the launch csv to profiles/TAG_launches.csv.
"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
out_md = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", f"{tag}_ncu.md")
src = os.path.join(ROOT, "gpurun_out")

KEYS = [
    ("gpu__time_duration.sum", "kernel duration"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.per_cycle_active", "active warps/SM"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__inst_executed.sum", "warp instructions"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (warp-instr/clk/SM)"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue slots busy %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU pipe %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts % of peak"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes"),
]
STALLS = "smsp__average_warps_issue_stalled_"


def launches(path):
    rows = list(csv.reader(open(path)))
    i = next(n for n, r in enumerate(rows) if r and r[0] == "ID")
    h = rows[i]
    agg = collections.OrderedDict()
    for r in rows[i + 1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = d["Kernel Name"]
        short = name.split("(")[0].replace("void ", "")
        if "<" in short and not short.startswith("hs::"):
            short = short.split("<")[0]
        if short.startswith("hs::"):
            short = name.split("(hs::")[0].split("(int")[0].split("(long")[0].split("(const")[0].replace("void ", "")
        ns = float(d["Metric Value"]) * (1000.0 if d["Metric Unit"] == "us" else 1e6 if d["Metric Unit"] == "ms" else 1.0)
        e = agg.setdefault(short, [0, 0.0, d["Grid Size"], d["Block Size"]])
        e[0] += 1
        e[1] += ns
    return agg


def raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return [dict(zip(rows[0], zip(rows[1], r))) for r in rows[2:]]


lines = [f"# ncu summary `{tag}`", ""]
lp = os.path.join(src, f"{tag}_launches.csv")
if os.path.exists(lp):
    agg = launches(lp)
    tot = sum(v[1] for v in agg.values())
    ours = sum(v[1] for k, v in agg.items() if k.startswith("hs::"))
    lines += ["## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`)", "",
              "Cold-cache, serialised per-launch times; compare shares, not absolutes.", "",
              "| kernel | launches | grid | block | mean | total | share of all | share of hs:: |",
              "|---|---:|---|---|---:|---:|---:|---:|"]
    for k, (c, ns, g, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        share_h = f"{100 * ns / ours:.1f}%" if k.startswith("hs::") else ""
        lines.append(f"| `{k[:90]}` | {c} | {g} | {b} | {ns / c / 1e3:.1f} us | {ns / 1e6:.3f} ms | "
                     f"{100 * ns / tot:.1f}% | {share_h} |")
    lines.append("")
    shutil.copy(lp, os.path.join(ROOT, "profiles", f"{tag}_launches.csv"))
rp = os.path.join(src, f"{tag}.ncu-rep")
if os.path.exists(rp):
    for rec in raw(rp):
        name = rec.get("Kernel Name", ("?", "?"))[1]
        lines += [f"## Full capture (`ncu --set full --clock-control none`): `{name[:120]}`", "",
                  "| metric | value | unit |", "|---|---:|---|"]
        for key, label in KEYS:
            if key in rec:
                unit, val = rec[key]
                lines.append(f"| {label} (`{key}`) | {val} | {unit} |")
        st = []
        for key, (unit, val) in rec.items():
            if key.startswith(STALLS) and key.endswith("_per_issue_active.ratio") and "not_issued" not in key:
                try:
                    v = float(val)
                except ValueError:
                    continue
                if v >= 0.02:
                    st.append((v, key[len(STALLS):-len("_per_issue_active.ratio")]))
        lines += ["", "Warp stall reasons (cycles per issued instruction):", "",
                  "| reason | ratio |", "|---|---:|"]
        lines += [f"| {n} | {v:.3f} |" for v, n in sorted(st, reverse=True)]
        lines.append("")
        if ("eval_warp_kernel" in name or "eval8_kernel" in name) and os.environ.get("POP"):
            # per-launch DRAM traffic of the fitness kernel, read by bench.py
            # for roofline.traffic (bytes per launch at population POP)
            def num(key, scale):
                unit, val = rec[key]
                return float(val) * scale.get(unit, 1.0)
            byte_units = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            dram = num("dram__bytes_read.sum", byte_units) + num("dram__bytes_write.sum", byte_units)
            json.dump({"tag": tag, "kernel": name, "population": int(os.environ["POP"]),
                       "dram_bytes_per_launch": dram,
                       "smem_wavefronts_per_launch": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", {}),
                       "warp_instructions_per_launch": num("smsp__inst_executed.sum", {}) if "smsp__inst_executed.sum" in rec else None,
                       "duration_ms": num("gpu__time_duration.sum", {"ms": 1.0, "us": 1e-3, "ns": 1e-6}),
                       "alu_pipe_pct": num("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", {}),
                       "issue_active_pct": num("sm__issue_active.avg.pct_of_peak_sustained_elapsed", {}),
                       "ipc": num("sm__inst_executed.avg.per_cycle_active", {}),
                       "smem_pipe_pct": num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", {}),
                       "source": f"profiles/{tag}_ncu.md (ncu --set full --clock-control none, one launch)"},
                      open(os.path.join(ROOT, "profiles", "eval_traffic.json"), "w"), indent=1)
os.makedirs(os.path.dirname(out_md), exist_ok=True)
open(out_md, "w").write("\n".join(lines) + "\n")
print(out_md)
