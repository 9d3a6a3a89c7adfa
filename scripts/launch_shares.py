"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel name.
   python scripts/launch_shares.py gpurun_out/launches.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
iN, iV, iU = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
for r in rows[start + 1:]:
    if len(r) <= iV:
        continue
    a = agg[r[iN][:60]]
    a[0] += 1
    a[1] += float(r[iV].replace(",", "")) * scale.get(r[iU], 1.0)
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':60s} launches   total_ms   share")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:60s} {v[0]:8d} {v[1]:10.2f} {100 * v[1] / tot:6.1f}%")
