#!/usr/bin/env python3
"""Top SASS stall hotspots of an ncu report's source page:
    ncu -i rep.ncu-rep --page source --csv > src.csv; python tools/sass_hot.py src.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
ix = {name: i for i, name in enumerate(h)}
body = [r for r in rows[hi + 1:] if len(r) == len(h)]
S = ix["# Samples"]
tot = sum(float(r[S] or 0) for r in body)
ex = sum(float(r[ix["Instructions Executed"]] or 0) for r in body)
print("samples", tot, "warp instructions", ex, "SASS lines", len(body))
stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
agg = {c: sum(float(r[ix[c]] or 0) for r in body) for c in stalls}
print("by reason:", ", ".join(f"{c[6:]} {100 * v / tot:.1f}%" for c, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
order = sorted(range(len(body)), key=lambda i: -float(body[i][S] or 0))[:n]
for i in order:
    r = body[i]
    why = sorted(((float(r[ix[c]] or 0), c[6:]) for c in stalls), reverse=True)[:2]
    print(f"{i:5d} {float(r[S]):8.0f} {100 * float(r[S]) / tot:5.1f}% ex={r[ix['Instructions Executed']]:>9} "
          f"{r[ix['Source']][:70]:70s} {why[0][1]}:{why[0][0]:.0f} {why[1][1]}:{why[1][0]:.0f}")
