"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV).

usage: python profiles/launch_summary.py gpurun_out/launches.csv
"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h, data = rows[hi], rows[hi + 1:]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
mult = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in data:
    if len(r) <= vi:
        continue
    name = r[ki]
    m = re.search(r"\b(k_[a-z_0-9]+(<[a-z0-9]+>)?)", name)
    if m:
        short = m.group(1)
    else:
        m = re.search(r"(Device\w+Kernel|\w+Kernel)", name)
        short = ("cub::" + m.group(1)) if m else name[:60]
    agg[short][0] += 1
    agg[short][1] += float(r[vi].replace(",", "")) * mult[r[ui]]
tot = sum(a[1] for a in agg.values())
print(f"{'us total':>10} {'n':>4} {'us/launch':>10} {'share':>6}  kernel")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:10.1f} {n:4d} {t / n:10.1f} {100 * t / tot:5.1f}%  {k}")
print(f"total {tot:.1f} us")
