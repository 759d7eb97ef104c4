#!/usr/bin/env python3
"""Cost of cutting a stage into element chunks (the e2e wavefront's launches): one
full-range volume / interface launch vs C range launches over the same elements."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_02516_b200 import capi  # noqa: E402

k1d = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
case = capi.Case("smooth", N=4, nx=k1d, warp=0.1, seed=23)
h = case.handle()
st = torch.cuda.Stream()
h.set_stream(st.cuda_stream)
h.set_state(case.u0())
h.step(case.dt, 2)
K = case.K
dt = case.dt


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for C in (1, 4, 16, 32):
    bounds = [K * i // C // 2 * 2 for i in range(C)] + [K]
    vol = timed(lambda: [h.stage_volume_range(1, dt, bounds[i], bounds[i + 1]) for i in range(C)])
    srf = timed(lambda: [h.stage_surface_range(1, dt, bounds[i], bounds[i + 1]) for i in range(C)])
    print(f"chunks {C:3d}: volume {vol:.3f} ms, interface {srf:.3f} ms", flush=True)
h.check()
