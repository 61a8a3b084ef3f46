"""Aggregate an ncu report's SASS metrics per CUDA source line (File, Line).

usage: python tools/ncu_srclines.py REPORT KERNEL_REGEX [units] [min_frac]
units: divide instruction counts by this (e.g. samples) for per-unit figures.
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
units = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
minf = float(sys.argv[4]) if len(sys.argv) > 4 else 0.005
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
agg = {}
fname, hdr = None, None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        ie, st = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
        continue
    # source-line rows carry the aggregate over their SASS; SASS rows have an empty line number
    if hdr is None or not r[0] or len(r) <= ie or r[ie] in ("", "-"):
        continue
    try:  # ncu does not escape quotes inside inline-asm source lines: skip those rows
        key = (fname, int(r[0]), r[1].strip()[:90])
        n, s = int(r[ie]), (int(r[st]) if r[st] not in ("", "-") else 0)
    except ValueError:
        continue
    a = agg.setdefault(key, [0, 0])
    a[0] += n
    a[1] += s
tot = sum(v[0] for v in agg.values())
stot = sum(v[1] for v in agg.values()) or 1
print(f"total {tot / units:.1f} warp-instr per unit")
for (f, ln, src), (n, s) in sorted(agg.items(), key=lambda kv: (kv[0][0], kv[0][1])):
    if n > tot * minf or s > stot * 0.01:
        print(f"{f}:{ln:<4} {n / units:8.1f} {n / tot * 100:5.1f}% stall {s / stot * 100:5.1f}%  {src}")
