"""Aggregate an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel name.
usage: python tools/launch_summary.py launches.csv [top]"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr, agg = None, defaultdict(lambda: [0, 0.0])
scale = {"ns": 1e-3, "nsecond": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    us = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], float("nan"))
    k = d["Kernel Name"].split("(")[0][:80]
    agg[k][0] += 1
    agg[k][1] += us
tot = sum(v[1] for v in agg.values())
print(f"total {tot:.1f} us over {sum(v[0] for v in agg.values())} launches")
for k, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{c:6d} {us:12.1f} us {us / c:10.2f} us/launch  {100 * us / tot:5.1f}%  {k}")
