#!/usr/bin/env python3
"""C3 (SBP N=4 dam break, K1D=128) step loop for profiling: python tools/sbp_probe.py [K1D] [steps]."""
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2005_02516_b200 import capi  # noqa: E402

k1d = int(sys.argv[1]) if len(sys.argv) > 1 else 128
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
c = capi.Case("dambreak", scheme=capi.SCHEME_SBP, N=4, nx=k1d, cfl=0.0625)
h = c.handle(mode=capi.MODE_FAST)
h.set_state(c.u0())
h.set_graphs(False)
h.step(c.dt, steps)
print("ok", c.K)
