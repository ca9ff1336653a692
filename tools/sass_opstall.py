"""Stall-reason samples per opcode class (ncu source page)."""
import csv, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
si = h.index('Source')
cols = [c for c in h if c.startswith('stall_') and '(' not in c]
agg = defaultdict(lambda: defaultdict(int))
for r in rows[1:]:
    if len(r) < len(h):
        continue
    t = r[si].split()
    op = (t[1] if t and t[0].startswith('@') else (t[0] if t else '?')).split('.')[0]
    for c in cols:
        agg[op][c] += int(r[h.index(c)] or 0)
tot = sum(sum(d.values()) for d in agg.values())
for op, d in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:8]:
    s = sum(d.values())
    top = sorted(d.items(), key=lambda kv: -kv[1])[:6]
    print(f"{op:8s} {100*s/tot:5.1f}%  " + "  ".join(f"{k[6:]}={100*v/tot:.1f}" for k, v in top))
