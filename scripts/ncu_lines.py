#!/usr/bin/env python3
"""Attribute ncu per-SASS metrics to CUDA source lines.

usage: ncu_lines.py REPORT.ncu-rep KERNEL_MANGLED_SUBSTR LIB.so [topN]
Uses `ncu --page source --print-source=sass` for per-address metrics and
`nvdisasm -g` on the library's cubins for address -> file:line.
"""
import csv, os, re, subprocess, sys, tempfile, collections

rep, kern, lib = sys.argv[1:4]
lib = os.path.abspath(lib)
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
addr2line = {}
for f in os.listdir(tmp):
    if not f.endswith(".cubin"):
        continue
    txt = subprocess.run(["nvdisasm", "-g", "-c", f], cwd=tmp, capture_output=True, text=True).stdout
    infn = False
    cur = None
    for ln in txt.splitlines():
        if ln.startswith("//---") and ".text." in ln:
            infn = kern in ln
            continue
        if not infn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            if "inlined at" not in ln:
                cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            else:
                cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            addr2line[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, *os.environ.get("NCU_FILTER", "").split(), "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = None
base = None
for r in rows:
    if r and r[0].startswith("0x"):
        v = int(r[0], 16)
        base = v if base is None else min(base, v)
agg = collections.defaultdict(lambda: collections.Counter())
tot = collections.Counter()
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    try:
        a = int(d["Address"], 16) - base
    except ValueError:
        continue
    line = addr2line.get(a, "?")
    for k in ("Instructions Executed", "Warp Stall Sampling (All Samples)", "Thread Instructions Executed",
              "L1 Wavefronts Shared"):
        try:
            v = float(d.get(k, 0) or 0)
        except ValueError:
            v = 0
        agg[line][k] += v
        tot[k] += v
print(f"{'line':28s} {'inst%':>6s} {'stall%':>6s} {'thr/inst':>8s} {'smemwf%':>7s}")
for line, c in sorted(agg.items(), key=lambda kv: -kv[1]["Warp Stall Sampling (All Samples)"])[:top]:
    ie = c["Instructions Executed"]
    print(f"{line:28s} {100*ie/max(tot['Instructions Executed'],1):6.1f} "
          f"{100*c['Warp Stall Sampling (All Samples)']/max(tot['Warp Stall Sampling (All Samples)'],1):6.1f} "
          f"{c['Thread Instructions Executed']/max(ie,1):8.1f} "
          f"{100*c['L1 Wavefronts Shared']/max(tot['L1 Wavefronts Shared'],1):7.1f}")
