"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]; ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value")
d = defaultdict(list)
for r in rows[1:]:
    d[r[ki].split("(")[0][:60]].append(float(r[vi]))
tot = sum(sum(v) for v in d.values())
for k, v in sorted(d.items(), key=lambda x: -sum(x[1])):
    print(f"{k:60s} n={len(v):4d} mean={sum(v)/len(v)/1e3:9.2f} us share={sum(v)/tot:.4f}")
