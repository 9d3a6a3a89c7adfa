"""Print the hottest SASS regions of an ncu report (source page, sass view)."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 60
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
iS, iI, iSrc, iT = h.index('Warp Stall Sampling (All Samples)'), h.index('Instructions Executed'), h.index('Source'), h.index('Thread Instructions Executed')
data = [(int(r[iS] or 0), int(r[iI] or 0), int(r[iT] or 0), r[0], r[iSrc].strip()) for r in rows[2:] if len(r) > iI]
tot_s = sum(d[0] for d in data); tot_i = sum(d[1] for d in data)
print(f'total samples {tot_s}, total warp insts {tot_i}')
mode = sys.argv[3] if len(sys.argv) > 3 else 'listing'
if mode == 'listing':
    for s, i, t, a, src in data:
        if i > tot_i * 0.0005 or s > tot_s * 0.002:
            print(f'{a[-5:]} {100*s/tot_s:5.1f}% {i:12d} {t/max(i,1):5.1f} {src}')
