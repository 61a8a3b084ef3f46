"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list per kernel (ms, count)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ik, iv = h.index("Kernel Name"), h.index("Metric Value")
iu = h.index("Metric Unit") if "Metric Unit" in h else None
agg, cnt = collections.OrderedDict(), collections.Counter()
for r in rows[hi + 1:]:
    if len(r) <= iv:
        continue
    k = r[ik].split("(")[0][:70]
    v = float(r[iv].replace(",", ""))
    u = r[iu] if iu is not None else "ns"
    v = v / 1e6 if u == "ns" else v / 1e3 if u == "us" else v
    agg[k] = agg.get(k, 0.0) + v
    cnt[k] += 1
for k, v in sorted(agg.items(), key=lambda x: -x[1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{v:9.2f} ms  x{cnt[k]:4d}  {k}")
print(f"total {sum(agg.values()):.2f} ms")
