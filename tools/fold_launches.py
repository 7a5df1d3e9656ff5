"""Aggregate an ncu launch-list CSV (gpu__time_duration.sum [+ dram bytes]) per kernel.

    python tools/fold_launches.py launches.csv [--last-half]
"""
import csv
import sys
from collections import OrderedDict, defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10][1:]
k = OrderedDict()
for r in rows:
    k.setdefault(r[0], {"name": r[4].split("(")[0][:80]})[r[-3]] = float(r[-1].replace(",", ""))
ids = list(k.keys())
if "--last-half" in sys.argv:
    ids = ids[len(ids) // 2:]
agg = defaultdict(lambda: [0, 0.0, 0.0])
for i in ids:
    d = k[i]
    a = agg[d["name"]]
    a[0] += 1
    a[1] += d.get("gpu__time_duration.sum", 0) / 1e6
    a[2] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
tot = sum(v[1] for v in agg.values())
print(f"total {tot:.3f} ms over {len(ids)} launches")
for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1])[:25]:
    gbs = b / 1e9 / (t / 1e3) if t else 0.0
    print(f"{t:8.3f} ms {100 * t / tot:5.1f}% {c:4d}x {b / 1e6:9.1f} MB {gbs:8.1f} GB/s  {n}")
