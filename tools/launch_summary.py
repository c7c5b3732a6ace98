#!/usr/bin/env python
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: count, total and average
device time per kernel and each kernel's share (cold-cache, serialised times: compare shares)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[h]
agg = collections.OrderedDict()
for r in rows[h + 1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    unit = d["Metric Unit"]
    v = float(d["Metric Value"].replace(",", "")) * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
print(f"{'launches':>8} {'total_us':>12} {'avg_us':>10} {'share':>7}  kernel")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{n:8d} {t:12.1f} {t / n:10.1f} {t / tot:7.1%}  {k}")
print(f"{sum(a[0] for a in agg.values()):8d} {tot:12.1f}")
