"""Per-CUDA-source-line instruction and stall-sample shares of an ncu report (cuda,sass view).

   python scripts/ncu_lines.py gpurun_out/k4.ncu-rep [top]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file = ""
agg = {}
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("Function Name",):
        continue
    if r[2] != "-":  # sass rows carry an address in column 2; cuda rows have '-'
        continue
    try:
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        iI = hdr.index("Instructions Executed")
        s, i = int(r[iS] or 0), int(r[iI] or 0)
    except (ValueError, IndexError):
        continue
    key = (cur_file, int(r[0]), r[1].strip()[:90])
    a = agg.setdefault(key, [0, 0])
    a[0] += s
    a[1] += i
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"{'file:line':28s} {'%inst':>6s} {'%samp':>6s}  source")
for (f, ln, src), (s, i) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{f + ':' + str(ln):28s} {100 * i / ti:6.1f} {100 * s / ts:6.1f}  {src}")
