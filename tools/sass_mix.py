"""Instruction mix of a profiled kernel from `ncu --page source --print-source sass`:
executed warp instructions per opcode and the stall samples they carry."""
import csv, subprocess, sys
from collections import Counter
rep = sys.argv[1]
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
si, ei, ss = h.index('Source'), h.index('Instructions Executed'), h.index('Warp Stall Sampling (All Samples)')
ops, stalls = Counter(), Counter()
tot = 0
for r in rows[1:]:
    if len(r) <= ei:
        continue
    op = r[si].split()[0] if r[si].split() else '?'
    if op.startswith('@'):
        op = r[si].split()[1]
    op = op.split('.')[0]
    n = int(r[ei] or 0)
    ops[op] += n
    stalls[op] += int(r[ss] or 0)
    tot += n
st = sum(stalls.values())
for op, n in ops.most_common(25):
    print(f"{op:10s} {n:14d} {100*n/tot:6.2f}%   stall samples {100*stalls[op]/max(st,1):6.2f}%")
print('total', tot)
