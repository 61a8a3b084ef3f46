"""Print the shared-memory pipeline and issue metrics of each kernel in ncu reports."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum", "smsp__inst_executed_op_shared_atom.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "dram__bytes_read.sum",
        "smsp__inst_executed_op_shfl.sum", "l1tex__data_pipe_lsu_wavefronts.sum"]
for rep in sys.argv[1:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    for r in rows[2:]:
        d = dict(zip(rows[0], r))
        print("==", rep, d["Kernel Name"][:60])
        for k in KEYS:
            print(f"  {k:70s} {d.get(k)}")
