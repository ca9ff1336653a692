"""Top SASS lines of a profiled kernel by one stall reason (ncu source page)."""
import csv, subprocess, sys
rep, col = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(['ncu', '-i', rep, '--page', 'source', '--csv', '--print-source', 'sass'],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
ci, si, ai, ei = h.index(col), h.index('Source'), h.index('Address'), h.index('Instructions Executed')
body = [r for r in rows[1:] if len(r) > ci]
tot = sum(int(r[ci] or 0) for r in body)
idx = {r[ai]: i for i, r in enumerate(body)}
for r in sorted(body, key=lambda r: -int(r[ci] or 0))[:n]:
    print(f"{int(r[ci]):8d} {100*int(r[ci])/max(tot,1):5.1f}%  #{idx[r[ai]]:5d} exec {int(r[ei] or 0):11d}  {r[si].strip()[:70]}")
print('total', tot)
