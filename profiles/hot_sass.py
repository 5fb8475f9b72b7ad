#!/usr/bin/env python3
"""Summarise an `ncu --page source --csv` dump: hottest SASS lines by executed warp instructions."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
thresh = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iex, ist = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[hi + 1:] if len(r) > max(iex, ist)]
tot = sum(int(r[iex]) for r in data if r[iex].isdigit())
stall = sum(int(r[ist]) for r in data if r[ist].isdigit())
print("total warp instr", tot, "stall samples", stall, "lines", len(data))
for r in data:
    n = int(r[iex]) if r[iex].isdigit() else 0
    s = int(r[ist]) if r[ist].isdigit() else 0
    if n > tot * thresh / 100 or s > stall * thresh / 100:
        print(f"{r[ia][-5:]} ex={n / tot * 100:5.2f}% stall={s / max(stall, 1) * 100:5.2f}%  {r[isrc][:100]}")
