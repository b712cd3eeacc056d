"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
d = defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > vi:
        d[r[ki][:70]].append(float(r[vi].replace(",", "")))
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
tot = 0.0
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    v = v[skip:] if len(v) > skip else v
    tot += sum(v) / len(v) if len(v) > 2 else 0
    print(f"{len(v):5d} {sum(v) / len(v) / 1000:9.2f} us  {k}")
