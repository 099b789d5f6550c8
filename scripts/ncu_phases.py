#!/usr/bin/env python3
"""Per-phase (source file / line range) and per-opcode split of an ncu
source-page capture: warp instructions, stall samples and shared-memory
wavefronts (actual vs ideal) per evaluated layout.

usage: ncu_phases.py REPORT.ncu-rep KERNEL_SUBSTR LIB.so UNITS
"""
import collections, csv, os, re, subprocess, sys, tempfile

rep, kern, lib, units = sys.argv[1], sys.argv[2], os.path.abspath(sys.argv[3]), float(sys.argv[4])
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
a2l = {}
for f in os.listdir(tmp):
    if not f.endswith(".cubin"):
        continue
    txt = subprocess.run(["nvdisasm", "-g", "-c", f], cwd=tmp, capture_output=True, text=True).stdout
    infn, cur = False, None
    for ln in txt.splitlines():
        if ln.startswith("//---") and ".text." in ln:
            infn = kern in ln
            continue
        if not infn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            a2l[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr, base = None, None
for r in rows:
    if r and r[0].startswith("0x"):
        v = int(r[0], 16)
        base = v if base is None else min(base, v)
K = ("Instructions Executed", "Warp Stall Sampling (All Samples)", "L1 Wavefronts Shared",
     "L1 Wavefronts Shared Ideal")
byf, byop = collections.defaultdict(collections.Counter), collections.defaultdict(collections.Counter)
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
    fil = a2l.get(a, "?").split(":")[0]
    op = d["Source"].split()[0] if d["Source"].split() else "?"
    if op.startswith("@"):
        op = d["Source"].split()[1]
    op = op.split(".")[0]
    for k in K:
        v = float(d.get(k, 0) or 0)
        byf[fil][k] += v
        byop[(fil, op)][k] += v
        tot[k] += v
print(f"{'file':24s} {'op':10s} {'winst/u':>8s} {'inst%':>6s} {'stall%':>6s} {'wf/u':>7s} {'ideal/u':>8s}")
for f, c in sorted(byf.items(), key=lambda kv: -kv[1][K[0]]):
    print(f"{f:24s} {'':10s} {c[K[0]]/units:8.1f} {100*c[K[0]]/tot[K[0]]:6.1f} {100*c[K[1]]/tot[K[1]]:6.1f} "
          f"{c[K[2]]/units:7.1f} {c[K[3]]/units:8.1f}")
    for (f2, op), c2 in sorted(byop.items(), key=lambda kv: -kv[1][K[0]]):
        if f2 != f or c2[K[0]] / units < 4:
            continue
        print(f"{'':24s} {op:10s} {c2[K[0]]/units:8.1f} {100*c2[K[0]]/tot[K[0]]:6.1f} {100*c2[K[1]]/tot[K[1]]:6.1f} "
              f"{c2[K[2]]/units:7.1f} {c2[K[3]]/units:8.1f}")
print(f"total warp-instr/unit {tot[K[0]]/units:.1f}, smem wavefronts/unit {tot[K[2]]/units:.1f} "
      f"(ideal {tot[K[3]]/units:.1f})")
