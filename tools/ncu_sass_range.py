#!/usr/bin/env python
"""Print the SASS of an address range (offsets from the kernel start) with
execution counts and stall samples.  Usage: ncu_sass_range.py SOURCE_CSV LO HI
(SOURCE_CSV = ncu -i REP --page source --csv --print-source=sass)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
ad, src, ie, ss = (h.index(k) for k in ("Address", "Source", "Instructions Executed", "Warp Stall Sampling (All Samples)"))
base = int(data[0][ad], 16)
lo, hi = int(sys.argv[2]), int(sys.argv[3])
for r in data:
    off = int(r[ad], 16) - base
    if lo <= off <= hi:
        print(f"{off:6d} {r[ie]:>10} {r[ss]:>6} {r[src].strip()}")
