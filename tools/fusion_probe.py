#!/usr/bin/env python3
"""Device-resident LSRK45 step time with the fused stage chain on/off (C4 workload)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_02516_b200 import capi  # noqa: E402

k1d = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
case = capi.Case("smooth", N=4, nx=k1d, warp=0.1, seed=23)
for fused in ("1", "0", "1"):
    os.environ["SWEDG_FUSION"] = fused
    h = case.handle()
    st = torch.cuda.Stream()
    h.set_stream(st.cuda_stream)
    h.set_state(case.u0())
    h.step(case.dt, 3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    h.step(case.dt, 10, sync=False)
    e1.record(st)
    torch.cuda.synchronize()
    h.check()
    print(f"fusion={fused}: {e0.elapsed_time(e1) / 10:.3f} ms/step", flush=True)
    h.close()
