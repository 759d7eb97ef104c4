#!/usr/bin/env python3
"""Attribute an ncu SASS source export to CUDA source lines: join the export's
per-instruction samples / executions / shared wavefronts with `nvdisasm -g` line info of
the same build (addresses relative to the kernel's first instruction).

    ncu -i rep --page source --csv --print-source sass -k regex:NAME > x.csv
    nvdisasm -g lib.sm_100a.cubin > all.sass        (cuobjdump -xelf all libswedg_b200.so)
    python tools/sass_lines.py x.csv all.sass KERNEL_MANGLED_SUBSTRING units [ntop]
"""
import csv
import re
import sys
from collections import defaultdict

csv_path, sass_path, kname, units = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
ntop = int(sys.argv[5]) if len(sys.argv) > 5 else 40
addr_line, infn, cur = {}, False, (None, None)
for ln in open(sass_path):
    if ln.startswith("\t.section") and ".text." in ln:
        infn = kname in ln
        continue
    if not infn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        addr_line[int(m.group(1), 16)] = (cur, m.group(2).strip())
rows = list(csv.reader(open(csv_path)))
hdr = [h.strip() for h in rows[1]]
ai, si, ei = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed")
sm = next(i for i, h in enumerate(hdr) if "All Samples" in h)
wf = hdr.index("L1 Wavefronts Shared")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[ai], 16), r[si].strip(), int(r[ei] or 0), int(r[sm] or 0), int(r[wf] or 0)))
    except (ValueError, IndexError):
        continue
base = min(d[0] for d in data)
per = defaultdict(lambda: [0, 0, 0, 0, 0])
ok = 0
for a, src, e, s, w in data:
    key = a - base
    if key not in addr_line:
        continue
    (f, l), txt = addr_line[key]
    ok += txt.split()[0] in src
    p = per[(f, l)]
    p[0] += s
    p[1] = max(p[1], e)
    p[2] += w
    p[3] += 1
    p[4] += any(x in src for x in ("DFMA", "DADD", "DMUL", "DMMA"))
print(f"instructions {len(data)}, mapped {sum(v[3] for v in per.values())}, opcode agreement {ok}")
T = sum(v[0] for v in per.values()) or 1
files = {}
for (f, l), (s, e, w, n, fp) in sorted(per.items(), key=lambda x: -x[1][0])[:ntop]:
    if f and f not in files:
        try:
            files[f] = open(f).read().splitlines()
        except OSError:
            files[f] = []
    text = files.get(f, [])[l - 1].strip()[:64] if f and l and l <= len(files.get(f, [])) else ""
    print(f"{100 * s / T:5.1f}%  exec {e:>9}  n {n:3d} fp64 {fp:3d}  wf/unit {w / units:6.1f}  "
          f"{(f or '?').split('/')[-1]}:{l}  {text}")
