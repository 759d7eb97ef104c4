#!/usr/bin/env python3
"""Summarise an ncu `--page source --csv --print-source sass` export: stall samples
grouped by execution count (loop nests) and the hottest instructions.

    ncu -i rep --page source --csv -k regex:NAME --print-source sass > x.csv
    python tools/sass_hot.py x.csv [ntop]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = [h.strip() for h in rows[1]]
si = hdr.index("Source")
wi = next(i for i, h in enumerate(hdr) if "All Samples" in h)
ei = hdr.index("Instructions Executed")
need = max(si, wi, ei)
data = [(int(r[wi] or 0), r[si].strip(), int(r[ei] or 0), i) for i, r in enumerate(rows[2:])
        if len(r) > need and (r[wi] or "0").isdigit() and (r[ei] or "0").isdigit()]
tot = sum(d[0] for d in data) or 1
print("total samples", tot, "instructions", len(data))
g = defaultdict(lambda: [0, 0, 0])
for s, src, e, _ in data:
    g[e][0] += s
    g[e][1] += 1
    g[e][2] += any(x in src for x in ("DFMA", "DADD", "DMUL"))
for e, (s, n, f) in sorted(g.items(), key=lambda x: -x[1][0])[:10]:
    print(f"exec {e:>10} ninstr {n:5d} fp64 {f:5d} samples {s:7d} {100 * s / tot:5.1f}%")
for d in sorted(data, key=lambda d: -d[0])[:ntop]:
    print(d[0], d[2], d[3], d[1][:100])
