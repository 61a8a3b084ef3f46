"""Per-kernel summary of an ncu --set full report as JSON (the numbers DESIGN.md quotes).

usage: python tools/ncu_summary.py REPORT.ncu-rep UNITS_PER_LAUNCH "CONFIG" > profiles/<wl>_ncu_full.json
CONFIG names the capture, e.g. "c3 n=2^24 p=1024 m=51 f32"; bench.py uses traffic_bytes only
when CONFIG's n matches the bench size.
"""
import csv
import io
import json
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
config = sys.argv[3] if len(sys.argv) > 3 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
keys = {
    "time_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_GB": ("dram__bytes_read.sum", None),
    "dram_write_GB": ("dram__bytes_write.sum", None),
    "warp_instructions": ("smsp__inst_executed.sum", 1.0),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "shared_atomics": ("smsp__inst_executed_op_shared_atom.sum", 1.0),
    # the shared-memory / L1 pipe: K3's binding resource (wavefronts; ATOMS ~2 LDS-equivalents)
    "l1tex_busy_pct": ("l1tex__throughput.avg.pct_of_peak_sustained_active", 1.0),
    "smem_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1.0),
    "smem_atom_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum", 1.0),
    "smem_ld_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", 1.0),
}
units_row = rows[1]
out = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    u = dict(zip(hdr, units_row))
    e = {"kernel": d["Kernel Name"][:80]}
    for k, (m, scale) in keys.items():
        if m not in d:
            continue
        v = float(d[m].replace(",", ""))
        if k == "time_ms":
            unit = u.get(m, "")
            v = v * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3,
                     "second": 1e3}[unit]
        elif scale is None:
            unit = u.get(m, "")
            v = v * {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}[unit]
        e[k] = v
    if "warp_instructions" in e:
        e["warp_instructions_per_unit"] = e["warp_instructions"] / units
    if "dram_read_GB" in e and "dram_write_GB" in e:
        e["traffic_bytes"] = (e["dram_read_GB"] + e["dram_write_GB"]) * 1e9
    out.append(e)
kernels = {}
for e in out:
    name = e.pop("kernel").replace("void ", "").replace("skc::", "")
    kernels.setdefault(name, e)
print(json.dumps({"config": config, "source": f"ncu --set full --clock-control none ({rep})",
                  "units_per_launch": units, "kernels": kernels}, indent=1))
