#!/usr/bin/env python
"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import re
import sys


def summarise(path, top=30):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        m = re.search(r"(k_\w+|at::\w+|\w+_kernel\w*)(<[^>]*>)?", r[ki])
        name = m.group(0) if m else r[ki][:50]
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    out = [f"{'kernel':44s} {'launches':>8s} {'total_ms':>10s} {'avg_us':>10s} {'share':>6s}"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        out.append(f"{k[:44]:44s} {v[0]:8d} {v[1] / 1e3:10.3f} {v[1] / v[0]:10.1f} {v[1] / tot * 100:5.1f}%")
    out.append(f"{'TOTAL':44s} {sum(v[0] for v in agg.values()):8d} {tot / 1e3:10.3f}")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1]))
