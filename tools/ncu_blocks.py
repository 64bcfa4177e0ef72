#!/usr/bin/env python
"""Basic blocks of the hottest kernel in an ncu report with their dynamic
instruction share (needs --import-source / SASS counts).
Usage: python tools/ncu_blocks.py REPORT [unit_count] [min_share]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
unit = float(sys.argv[2]) if len(sys.argv) > 2 else 0
thr = float(sys.argv[3]) if len(sys.argv) > 3 else 0.004
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Address")
data = [r for r in rows[rows.index(hdr) + 1:] if r and r[0].startswith("0x")]
ia = hdr.index("Instructions Executed")
base = int(data[0][0], 16)
seq = [(int(r[0], 16) - base, r[1].strip(), int(r[ia])) for r in data if r[ia].isdigit()]
tot = sum(x[2] for x in seq)
print(f"instructions {tot:.4e}" + (f"  per unit {tot / unit:.1f}" if unit else ""))
blocks, cur = [], None
for off, src, n in seq:
    if cur and cur[2] == n:
        cur[1] = off
        cur[3] += 1
    else:
        if cur:
            blocks.append(cur)
        cur = [off, off, n, 1, src]
blocks.append(cur)
for b in blocks:
    if b[2] * b[3] > tot * thr:
        extra = f"  per unit {b[2] * b[3] / unit:6.1f}" if unit else ""
        print(f"{b[0]:#7x}-{b[1]:#7x} count {b[2]:>11} x{b[3]:>4} = {100 * b[2] * b[3] / tot:5.1f}%{extra}  {b[4][:50]}")
