#!/usr/bin/env python3
"""e2e decomposition at C4: device-resident steps (graph replay), the chunked host-state
wavefront, and (with a -DSWEDG_E2E_NOCOPY build via SWEDG_LIB_VARIANT) the wavefront's
launches without the copies.  ms per step, 10 steps after a warm-up call."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_02516_b200 import capi  # noqa: E402

case = capi.Case("smooth", N=4, nx=1024, warp=0.1, seed=23)
u0 = case.u0()
h = case.handle(diagnostics=False)
st = torch.cuda.Stream()
h.set_stream(st.cuda_stream)
uh = torch.empty(u0.shape, dtype=torch.float64, pin_memory=True).numpy()


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 10


h.set_state(u0)
h.step(case.dt, 3)
print(f"device-resident (graph): {timed(lambda: h.step(case.dt, 10, sync=False)):.2f} ms/step", flush=True)
for C in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "16").split(",")]:
    uh[...] = u0
    h.set_state(uh)
    h.step_host(uh, case.dt, 1, C)
    print(f"host-state wavefront, {C} chunks: {timed(lambda: h.step_host(uh, case.dt, 10, C)):.2f} ms/step", flush=True)
