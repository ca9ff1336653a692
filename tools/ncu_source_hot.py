"""Hot spots of an `ncu --page source --csv` dump: per kernel section, samples
by SASS opcode and the top instructions with their dominant stall reason."""
import csv, sys, re
from collections import Counter
csv.field_size_limit(10**9)
rows = list(csv.reader(open(sys.argv[1])))
want = sys.argv[2] if len(sys.argv) > 2 else ""
topn = int(sys.argv[3]) if len(sys.argv) > 3 else 25
secs, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "hdr": None, "rows": []}
        secs.append(cur)
    elif cur is not None and r and r[0] == "Address":
        cur["hdr"] = r
    elif cur is not None and cur["hdr"] and len(r) == len(cur["hdr"]):
        cur["rows"].append(r)
for s in secs:
    if want and want not in s["name"]:
        continue
    h = s["hdr"]
    si, ci, ei = h.index("Source"), h.index("# Samples"), h.index("Instructions Executed")
    stall = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
    tot = sum(int(r[ci] or 0) for r in s["rows"])
    tex = sum(int(r[ei] or 0) for r in s["rows"])
    print("==", s["name"][:90], "samples", tot, "warp-instr", tex, "static", len(s["rows"]))
    byop, exop = Counter(), Counter()
    for r in s["rows"]:
        m = re.match(r"\s*(@!?U?P\d+\s+)?([A-Z0-9_]+)", r[si])
        op = m.group(2) if m else "?"
        byop[op] += int(r[ci] or 0)
        exop[op] += int(r[ei] or 0)
    print("  samples by opcode:", ", ".join(f"{k} {v} ({100*v/max(tot,1):.0f}%)" for k, v in byop.most_common(12)))
    print("  executed by opcode:", ", ".join(f"{k} {v} ({100*v/max(tex,1):.0f}%)" for k, v in exop.most_common(14)))
    st = Counter()
    for r in s["rows"]:
        for i in stall:
            st[h[i]] += int(r[i] or 0)
    print("  stalls:", ", ".join(f"{k[6:]} {v}" for k, v in st.most_common(8)))
    idx = sorted(range(len(s["rows"])), key=lambda i: -int(s["rows"][i][ci] or 0))[:topn]
    for i in sorted(idx):
        r = s["rows"][i]
        dom = max(stall, key=lambda j: int(r[j] or 0))
        print(f"  [{i:5d}] {int(r[ci]):5d} x{int(r[ei] or 0):8d} {h[dom][6:]:12s} {r[si].strip()[:90]}")
