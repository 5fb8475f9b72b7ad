#!/usr/bin/env python3
"""Top source lines of a kernel in an .ncu-rep by executed instructions and by stall samples
(ncu -i REP --page source --csv --print-source cuda,sass; needs -lineinfo and --import-source on)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'cuda,sass'],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file, hdr, lines = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == 'File Path':
        cur_file = r[1].split('/')[-1]
    elif r[0] == 'Line No':
        hdr = r
    elif hdr and r[0].strip().isdigit():
        def col(name):
            try:
                return int(r[hdr.index(name)])
            except (ValueError, IndexError):
                return 0
        lines.append((cur_file, int(r[0]), r[1].strip(), col('Instructions Executed'), col('# Samples'), col('L1 Wavefronts Shared')))
ti = sum(l[3] for l in lines) or 1
ts = sum(l[4] for l in lines) or 1
print(f'total warp instructions {ti}, samples {ts} (all kernels of the report; lines of a file shared by several kernels are summed)')
print('--- by instructions executed')
for l in sorted(lines, key=lambda x: -x[3])[:top]:
    print(f'{100*l[3]/ti:5.1f}% inst {100*l[4]/ts:5.1f}% smp  smem_wf {l[5]:>10d}  {l[0]}:{l[1]:<4d} {l[2][:110]}')
print('--- by stall samples')
for l in sorted(lines, key=lambda x: -x[4])[:top]:
    print(f'{100*l[3]/ti:5.1f}% inst {100*l[4]/ts:5.1f}% smp  smem_wf {l[5]:>10d}  {l[0]}:{l[1]:<4d} {l[2][:110]}')
