#!/usr/bin/env python
"""Format an `ncu --metrics gpu__time_duration.sum --csv` launch list as
'id kernel grid ns share'.  Usage: python tools/launch_list.py LAUNCHES.csv [HEADER...]"""
import csv
import sys


def main():
    rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
    rows = [r for r in rows if r[12] == "gpu__time_duration.sum"]
    tot = sum(float(r[14]) for r in rows)
    for h in sys.argv[2:]:
        print(h)
    print("id kernel grid ns share")
    for r in rows:
        print(f"{r[0]} {r[4][:70]} {r[8]} {r[14]} {100 * float(r[14]) / tot:.1f}%")


if __name__ == "__main__":
    main()
