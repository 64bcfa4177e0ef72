#!/usr/bin/env python
"""Summarise an ncu report: key metrics, stall reasons and the hottest SASS
windows.  Usage: python tools/ncu_summary.py REPORT.ncu-rep [--json OUT]"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__occupancy_limit_registers", "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "lts__t_bytes.sum", "l1tex__t_bytes.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "lts__t_sectors_srcunit_tex_op_read.sum", "smsp__cycles_active.avg",
]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    raw = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    out = {}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            out[k] = (vals[i], units[i])
            print(f"{k:70s} {vals[i]:>20s} {units[i]}")
    stalls = [(h, vals[i]) for i, h in enumerate(hdr)
              if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("_per_issue_active.ratio")]
    stalls = sorted(((float(v.replace(",", "")), h) for h, v in stalls if v not in ("", "n/a")), reverse=True)[:8]
    print("top stall reasons (avg cycles per issued instruction):")
    for v, h in stalls:
        print(f"   {h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):50s} {v:.2f}")
    sass = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv", "--print-source=sass"))))
    h = sass[1]
    data = sass[2:]
    ie, ss, src = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    num = lambda x: int(x) if x.isdigit() else 0  # noqa: E731
    tot = sum(num(r[ie]) for r in data) or 1
    stot = sum(num(r[ss]) for r in data) or 1
    print(f"SASS instructions executed: {tot}, stall samples {stot}")
    win = []
    W = 32
    for i in range(0, len(data), W):
        ch = data[i:i + W]
        win.append((sum(num(r[ss]) for r in ch), sum(num(r[ie]) for r in ch), i, ch[0][src].strip()[:50]))
    print("hottest windows (stall share, instruction share):")
    for s, n, i, t in sorted(win, reverse=True)[:10]:
        print(f"   @{i:5d} stall {100 * s / stot:5.1f}%  inst {100 * n / tot:5.1f}%  {t}")
    # per CUDA source line (needs -lineinfo + --import-source on)
    cs = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"))))
    lines = []
    hdr2 = None
    fname = ""
    for r in cs:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            hdr2 = r
        elif hdr2 and r and r[0]:
            try:
                lines.append((int(r[4]), int(r[7]), fname, r[0], r[1].strip()[:70]))
            except (ValueError, IndexError):
                pass
    if lines:
        ts = sum(x[0] for x in lines) or 1
        ti = sum(x[1] for x in lines) or 1
        print("hottest source lines (stall share, instruction share):")
        for s, n, f, ln, src_ in sorted(lines, reverse=True)[:25]:
            print(f"   {f}:{ln:>4s} stall {100 * s / ts:5.1f}%  inst {100 * n / ti:5.1f}%  {src_}")
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as f:
            json.dump({"metrics": out, "stalls": stalls, "inst_total": tot}, f, indent=1)


if __name__ == "__main__":
    main()
