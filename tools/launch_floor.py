#!/usr/bin/env python3
"""Per-launch floor of the stage kernels: time of a volume / interface launch over a
tiny element range (setup + one pair dominated), back to back."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_02516_b200 import capi  # noqa: E402

case = capi.Case("smooth", N=4, nx=256, warp=0.1, seed=23)
h = case.handle()
st = torch.cuda.Stream()
h.set_stream(st.cuda_stream)
h.set_state(case.u0())
h.step(case.dt, 1)
dt = case.dt
for n in (2, 4736, 2 * 4736):
    for name, fn in (("volume", lambda: h.stage_volume_range(1, dt, 0, n)),
                     ("interface", lambda: h.stage_surface_range(1, dt, 0, n))):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(50):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        print(f"{name} over {n} elements: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us per launch", flush=True)
h.check()
