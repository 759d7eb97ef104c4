#!/usr/bin/env python3
"""Device-resident LSRK45 step time (C4 workload) with graphs on/off; run with SWEDG_PDL=0/1."""
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
for graphs in (True, False, True):
    h.set_graphs(graphs)
    h.step(case.dt, 3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    h.step(case.dt, 10, sync=False)
    e1.record(st)
    torch.cuda.synchronize()
    h.check()
    print(f"PDL={os.environ.get('SWEDG_PDL', '1')} graphs={graphs}: {e0.elapsed_time(e1) / 10:.3f} ms/step", flush=True)
