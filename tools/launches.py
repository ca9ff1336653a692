"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv, sys
from collections import OrderedDict
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
tot = 0.0
for r in rows[hdr + 1:]:
    v = float(r[vi].replace(',', '')) / 1e3
    tot += v
    print(f"{r[ki].split('(')[0][:70]:72s} {v:10.1f} us")
print(f"{'total':72s} {tot:10.1f} us")
