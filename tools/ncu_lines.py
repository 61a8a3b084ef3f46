"""Summarise an ncu report: headline metrics and the hottest SASS lines of one kernel.

usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [min_frac]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
minf = float(sys.argv[3]) if len(sys.argv) > 3 else 0.004
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--kernel-name", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
d = dict(zip(rows[0], rows[2]))
for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
          "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed_op_shared_atom.sum",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]:
    print(f"{k:60s} {d.get(k, '?')}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
ie, sc, st, at = (h.index(x) for x in ("Instructions Executed", "Source", "Warp Stall Sampling (All Samples)",
                                       "Avg. Threads Executed"))
data = [(r[0], r[sc], int(r[ie] or 0), int(r[st] or 0), r[at]) for r in rows[2:] if len(r) > ie]
tot = sum(x[2] for x in data)
stot = sum(x[3] for x in data)
print("total warp-instructions", tot, "stall samples", stot)
for a, s, n, sl, avg in data:
    if n > tot * minf or sl > stot * 0.01:
        print(f"{a[-5:]} {n / tot * 100:5.2f}% stall {sl / stot * 100:5.2f}% thr {avg:>3} {s.strip()[:80]}")
