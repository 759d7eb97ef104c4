#!/usr/bin/env python3
"""e2e (host-state stepping) per-step time vs chunk count, 10 steps after a warm-up call."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_02516_b200 import capi  # noqa: E402

case = capi.Case("smooth", N=4, nx=1024, warp=0.1, seed=23)
u0 = case.u0()
h = case.handle()
st = torch.cuda.Stream()
h.set_stream(st.cuda_stream)
uh = torch.empty(u0.shape, dtype=torch.float64, pin_memory=True).numpy()
for C in [int(x) for x in (sys.argv[1].split(',') if len(sys.argv) > 1 else '4,6,8,12,16,24'.split(','))]:
    uh[...] = u0
    h.set_state(uh)
    h.step_host(uh, case.dt, 1, C)  # warm-up (adjacency check, events)
    uh[...] = u0
    h.set_state(uh)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    h.step_host(uh, case.dt, 10, C)
    e1.record(st)
    torch.cuda.synchronize()
    print(f"chunks {C}: {e0.elapsed_time(e1) / 10:.2f} ms/step", flush=True)
