#!/usr/bin/env python
"""Per-region instruction/stall breakdown of an ncu report's SASS page:
contiguous runs of instructions with the same execution count, largest first,
normalised per warp-row.  Usage: ncu_regions.py REPORT [rows_total] [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
rows_total = float(sys.argv[2]) if len(sys.argv) > 2 else 20 * 2048 * 8 * 512
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
ie, ss, src, ad = (h.index(k) for k in ("Instructions Executed", "Warp Stall Sampling (All Samples)", "Source",
                                         "Address"))
num = lambda x: int(x) if x.isdigit() else 0  # noqa: E731
base = int(data[0][ad], 16)
tot = sum(num(r[ss]) for r in data) or 1
itot = sum(num(r[ie]) for r in data)
print(f"instructions {itot}  per warp-row {itot / rows_total:.1f}")
reg = []
for r in data:
    off = int(r[ad], 16) - base
    n, s = num(r[ie]), num(r[ss])
    if reg and reg[-1][2] == n and off == reg[-1][1] + 16:
        reg[-1][1] = off
        reg[-1][3] += 1
        reg[-1][4] += s
    else:
        reg.append([off, off, n, 1, s])
agg = sorted(((x[2] * x[3], x) for x in reg if x[2] > 0), key=lambda t: -t[0])
for w, x in agg[:N]:
    print(f"{x[0]:6d}-{x[1]:6d} cnt {x[2]:>10d} ninst {x[3]:4d} per-row {w / rows_total:7.2f} stall {x[4] / tot * 100:5.2f}%")
