"""Print an ncu launch list (gpu__time_duration) in launch order for kernels matching a regex."""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
pat = re.compile(sys.argv[2] if len(sys.argv) > 2 else ".")
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
for r in rows[hi + 1:]:
    if len(r) > iv and pat.search(r[ik]):
        v = float(r[iv].replace(",", ""))
        v = v / 1e6 if r[iu] == "ns" else v / 1e3 if r[iu] == "us" else v
        print(f"{v:9.3f} ms  {r[ik].split('(')[0][:60]}")
