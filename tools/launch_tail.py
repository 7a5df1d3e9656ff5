"""Per-kernel device times of the last derive_plan step in an ncu launch list.

    python tools/launch_tail.py gpurun_out/c1_launches.csv [n_last]
"""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
last = int(sys.argv[2]) if len(sys.argv) > 2 else 8
tot = 0.0
for r in rows[-last:]:
    us = float(r[vi].replace(",", "")) / 1000
    tot += us
    print(f"  {r[ki][:60]:60s} {us:8.1f} us")
print(f"  {'sum':60s} {tot:8.1f} us")
