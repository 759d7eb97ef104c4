#!/usr/bin/env python3
"""Host-state wavefront stepping vs device-resident steps at C4: identical state, timing."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_02516_b200 import capi  # noqa: E402

case = capi.Case("smooth", N=4, nx=int(sys.argv[1]) if len(sys.argv) > 1 else 1024, warp=0.1, seed=23)
u0 = case.u0()
h = case.handle()
st = torch.cuda.Stream()
h.set_stream(st.cuda_stream)
uh = torch.empty(u0.shape, dtype=torch.float64, pin_memory=True).numpy()
for label in ("device graph", "device no-graph", "host wavefront"):
    uh[...] = u0
    h.set_state(uh)
    h.set_graphs(label == "device graph")
    torch.cuda.synchronize()
    t = time.perf_counter()
    if label.startswith("device"):
        h.step(case.dt, 6)
    else:
        h.step_host(uh, case.dt, 6, 16)
    torch.cuda.synchronize()
    el = time.perf_counter() - t
    u, _, tt = h.get_state(with_res=False)
    if label == "device graph":
        ref = u.copy()
    print(f"{label}: {el / 6 * 1e3:.2f} ms/step, t={tt}, equal to device: {np.array_equal(u, ref)}, "
          f"host copy equal: {np.array_equal(uh, u) if label.startswith('host') else '-'}", flush=True)
