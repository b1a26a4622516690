"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) per kernel: count, total, mean.
usage: python tools/launch_summary.py launches.csv [skip_first_n_launches]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
hdr = rows[0]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
agg = collections.OrderedDict()
for r in rows[1 + skip:]:
    name = r[ki].split("(")[0][:70]
    v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
print(f"total {tot:.1f} us over {sum(a[0] for a in agg.values())} launches")
for k, (n, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:6d} {v:12.1f} us {100 * v / tot:5.1f}% {v / n:10.1f} us/launch  {k}")
