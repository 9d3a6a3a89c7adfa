"""Per-instruction stall breakdown of the hottest SASS lines of an ncu report (source page).
usage: python scripts/ncu_stalls.py report.ncu-rep [min_exec_frac]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.002
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
cols = ['stall_wait', 'stall_short_sb', 'stall_math', 'stall_long_sb', 'stall_not_selected', 'stall_selected',
        'stall_branch_resolving', 'stall_dispatch', 'stall_mio']
ix = {c: h.index(c) for c in cols}
iI, iSrc, iS = h.index('Instructions Executed'), h.index('Source'), h.index('Warp Stall Sampling (All Samples)')
data = [r for r in rows[2:] if len(r) > iI]
tot_i = sum(int(r[iI] or 0) for r in data)
tot_s = sum(int(r[iS] or 0) for r in data)
print(f'samples {tot_s}  warp insts {tot_i}')
print('addr  ' + ' '.join(f'{c[6:12]:>7}' for c in cols) + '  source')
for r in data:
    if int(r[iI] or 0) > thr * tot_i:
        print(f'{r[0][-5:]} ' + ' '.join(f'{100 * int(r[ix[c]] or 0) / tot_s:7.2f}' for c in cols) + '  ' + r[iSrc].strip()[:60])
