#!/usr/bin/env python3
"""C3 (SBP N=4 dam break, 128x128) run toward T=1.5 in FAST and PARITY (bit-for-bit the
reference's arithmetic): reports how far each gets (positivity) and how far apart they are."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2005_02516_b200 import capi  # noqa: E402

nx = int(sys.argv[1]) if len(sys.argv) > 1 else 128
c = capi.Case("dambreak", scheme=capi.SCHEME_SBP, N=4, nx=nx, cfl=0.0625)
print(f"K={c.K} dt={c.dt:.4e}", flush=True)
for mode, name in ((capi.MODE_PARITY, "parity"), (capi.MODE_FAST, "fast")):
    h = c.handle(mode=mode)
    h.set_state(c.u0())
    t0 = time.time()
    n = 0
    minh = []
    try:
        while n * c.dt < 1.5:
            h.step(c.dt, 50)
            n += 50
            u, _, t = h.get_state()
            minh.append((round(t, 4), float(u[:, 0, :].min())))
    except capi.SwedgError as e:
        print(f"{name}: stopped after ~{n} steps: {e}", flush=True)
    print(f"{name}: wall {time.time() - t0:.1f}s, min h trace {minh[:8]} ... {minh[-3:]}", flush=True)
