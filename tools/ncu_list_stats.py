"""Median/min/max per kernel and metric of an ncu --csv launch list.
    python tools/ncu_list_stats.py list.csv"""
import csv, statistics, sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
d = defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    k = r[h.index("Kernel Name")].split("(")[0][:40]
    d[(k, r[h.index("Metric Name")])].append(float(r[h.index("Metric Value")].replace(",", "")))
for (k, m), v in sorted(d.items()):
    print(f"{k:40s} {m:30s} n={len(v):4d} med={statistics.median(v):12.1f} min={min(v):12.1f} max={max(v):12.1f}")
