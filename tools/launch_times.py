"""Mean duration per kernel from an ncu launch list (csv on stdin):
ncu --metrics gpu__time_duration.sum --clock-control none --csv CMD | python tools/launch_times.py"""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(sys.stdin) if len(r) > 10]
if rows:
    h = rows[0]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    acc = defaultdict(list)
    for r in rows[1:]:
        acc[r[ki].split("(")[0]].append(float(r[vi].replace(",", "")) / 1e3)
    for k, v in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k[:70]:70s} n={len(v):3d} mean={sum(v) / len(v):8.1f} us")
