"""Copy the judged evidence of one GPU round into profiles/ (tracked):
   launch-list shares (ncu gpu__time_duration, cold-cache serialised) and per-kernel
   `ncu --set full` metric summaries; k4_ncu_summary.json feeds bench.py's roofline.traffic.

   python scripts/summarize_profiles.py r01 [gpurun_out]
"""
import collections
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import summary  # noqa: E402

tag = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
dst = os.path.join(root, "profiles")
os.makedirs(dst, exist_ok=True)

# launch list
rows = list(csv.reader(open(os.path.join(src, "launches.csv"))))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[start]
iN, iV, iU = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}
for r in rows[start + 1:]:
    if len(r) <= iV:
        continue
    agg[r[iN].split("(")[0]][0] += 1
    agg[r[iN].split("(")[0]][1] += float(r[iV].replace(",", "")) * scale.get(r[iU], 1.0)
tot = sum(v[1] for v in agg.values())
with open(os.path.join(dst, f"{tag}_launch_shares.txt"), "w") as f:
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised):\n")
    f.write("# python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline (C3)\n")
    f.write(f"{'kernel':60s} {'launches':>8s} {'total_ms':>10s} {'share':>7s}\n")
    for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        f.write(f"{n:60s} {c:8d} {v:10.2f} {100 * v / tot:6.1f}%\n")
print(open(os.path.join(dst, f"{tag}_launch_shares.txt")).read())

for k in ("k4b", "k4a", "k4", "k1", "k2", "k3"):
    rep = os.path.join(src, f"{k}.ncu-rep")
    if not os.path.exists(rep):
        continue
    res = summary(rep)
    with open(os.path.join(dst, f"{tag}_{k}_ncu_full.txt"), "w") as f:
        f.write(f"# ncu --set full --clock-control none --import-source on -k regex:{k} -s 8 -c 1 (C3 bench)\n")
        for d in res:
            f.write(f"== {d.pop('kernel')}\n")
            for kk, v in d.items():
                f.write(f"   {kk:66s} {v}\n")
    if k == "k4b" or (k == "k4" and not os.path.exists(os.path.join(src, "k4b.ncu-rep"))):
        d = summary(rep)[0]
        rd = float(d["dram__bytes_read.sum"].split()[0]) * (1e6 if "Mbyte" in d["dram__bytes_read.sum"] else 1e9 if "Gbyte" in d["dram__bytes_read.sum"] else 1.0)
        wr = float(d["dram__bytes_write.sum"].split()[0]) * (1e6 if "Mbyte" in d["dram__bytes_write.sum"] else 1e9 if "Gbyte" in d["dram__bytes_write.sum"] else 1.0)
        fpl = int(os.environ.get("FRAMES_PER_LAUNCH", "219"))   # C3: ceil(262144 / 1200) frames per chunk
        json.dump({"tag": tag, "kernel": "k4b_blend" if k == "k4b" else "k4_composite", "config": "C3",
                   "dram_bytes_read": rd, "dram_bytes_write": wr, "frames_per_launch": fpl,
                   "dram_bytes_per_frame": (rd + wr) / fpl, "source": f"profiles/{tag}_{k}_ncu_full.txt"},
                  open(os.path.join(dst, "k4_ncu_summary.json"), "w"), indent=1)
    print("wrote", k)
