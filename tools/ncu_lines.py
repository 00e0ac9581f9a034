#!/usr/bin/env python
"""Per-source-line stall samples and executed instructions of one kernel in an ncu report
(needs -lineinfo and --import-source on): python tools/ncu_lines.py report.ncu-rep [units] [top]"""
import csv
import io
import subprocess
import sys


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


def main(path, units=1, top=40):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    agg = []
    for r in rows[3:]:
        if len(r) >= 8 and r[0] not in ("", "-"):
            agg.append([num(r[0]), r[1].strip()[:90], num(r[4]), num(r[7])])
    tot = sum(a[2] for a in agg) or 1
    print("stall samples", tot, "warp instructions", sum(a[3] for a in agg), "per unit", sum(a[3] for a in agg) / units)
    for a in sorted(agg, key=lambda x: -x[2])[:top]:
        print(f"{a[0]:5d} {a[2]:6d} {100 * a[2] / tot:5.1f}% {a[3] / units:9.1f}/unit  {a[1]}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 1, int(sys.argv[3]) if len(sys.argv) > 3 else 40)
