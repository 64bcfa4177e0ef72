#!/usr/bin/env python
"""Per-source-line instruction and stall shares of an ncu report (needs -lineinfo
and --import-source on).  Usage: python tools/ncu_lines.py REPORT [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
hdr, fname, lines = None, "", []
for r in csv.reader(io.StringIO(out)):
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and r and r[0]:
        try:
            lines.append((int(r[hdr.index("Instructions Executed")]), int(r[hdr.index("Warp Stall Sampling (All Samples)")]),
                          fname, r[0], r[1].strip()[:80]))
        except (ValueError, IndexError):
            pass
ti = sum(x[0] for x in lines) or 1
ts = sum(x[1] for x in lines) or 1
print(f"instructions {ti:.3e}  stall samples {ts}")
for n, s, f, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{100 * n / ti:5.1f}% inst {100 * s / ts:5.1f}% stall  {f}:{ln}  {src}")
