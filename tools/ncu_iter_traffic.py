"""Per-Lloyd-iteration DRAM traffic and time from an ncu launch list (host-driven loop).

usage: python tools/ncu_iter_traffic.py LAUNCHES.csv ITERATIONS POINTS "CONFIG" > profiles/<wl>_ncu_lloyd.json
LAUNCHES.csv: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv
of `SKC_LLOYD=host python tools/kmeans_iters.py <wl> ITERATIONS`. The per-iteration kernels are the
K-means ones launched once or more per iteration (assign, objective, partials, centres, reseed);
the once-per-sketch preparation (sketch, transposed sketch, K5t prep) is reported apart.
"""
import csv
import json
import re
import sys

path, iters, npts = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
config = sys.argv[4] if len(sys.argv) > 4 else ""
PREP = re.compile(r"indices_kernel|gather_tma|csc_|km_tc_bucket|km_tc_values|km_tc_entries|row_sqnorm|km_init|at::|cub::")
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
ik, im, iu, iv = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
ii = hdr.index("ID")
scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
         "ns": 1e-6, "us": 1e-3, "ms": 1.0}
launch = {}
for r in rows[1:]:
    d = launch.setdefault(r[ii], {"kernel": r[ik]})
    v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
    d[r[im]] = v
per = {}
prep = {}
for d in launch.values():
    name = re.sub(r"\(.*", "", d["kernel"]).replace("void ", "").replace("skc::", "")
    tgt = prep if PREP.search(d["kernel"]) else per
    e = tgt.setdefault(name, {"launches": 0, "time_ms": 0.0, "dram_bytes": 0.0})
    e["launches"] += 1
    e["time_ms"] += d.get("gpu__time_duration.sum", 0.0)
    e["dram_bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
tot_b = sum(e["dram_bytes"] for e in per.values()) / iters
tot_t = sum(e["time_ms"] for e in per.values()) / iters
print(json.dumps({"config": config, "source": f"ncu launch list ({path}), {iters} host-driven iterations",
                  "iterations": iters, "points": npts, "dram_bytes_per_iteration": tot_b,
                  "dram_bytes_per_point_iter": tot_b / npts, "kernel_ms_per_iteration": tot_t,
                  "per_iteration_kernels": {k: {kk: (vv / iters if kk != "launches" else vv) for kk, vv in e.items()}
                                            for k, e in sorted(per.items(), key=lambda x: -x[1]["time_ms"])},
                  "once_per_sketch": prep}, indent=1))
