#!/usr/bin/env python3
"""Device-resident LSRK45 throughput (GDOF*stages/s) vs mesh size and degree, FAST mode,
modal smooth-wave workload (the C4 generator) and SBP dam break (the C3 generator)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_02516_b200 import capi  # noqa: E402


def rate(case, steps):
    h = case.handle()
    st = torch.cuda.Stream()
    h.set_stream(st.cuda_stream)
    h.set_state(case.u0())
    h.step(case.dt, 3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    h.step(case.dt, steps, sync=False)
    e1.record(st)
    torch.cuda.synchronize()
    h.check()
    ms = e0.elapsed_time(e1) / steps
    dof = case.K * case.nstate * 3
    h.close()
    return ms, dof * 5 / (ms * 1e-3) / 1e9


for k1d in (64, 128, 256, 512, 1024, 2048):
    c = capi.Case("smooth", N=4, nx=k1d, warp=0.1, seed=23)
    ms, r = rate(c, 20 if k1d <= 1024 else 5)
    print(f"modal N=4 K1D={k1d:5d} K={c.K:8d}: {ms:8.3f} ms/step {r:7.2f} GDOF*stages/s", flush=True)
    c.close()
for N in (1, 2, 3):
    c = capi.Case("smooth", N=N, nx=512, warp=0.1, seed=23)
    ms, r = rate(c, 20)
    print(f"modal N={N} K1D=512 K={c.K}: {ms:.3f} ms/step {r:.2f} GDOF*stages/s", flush=True)
for k1d in (64, 128, 256, 512):
    c = capi.Case("dambreak", scheme=capi.SCHEME_SBP, N=4, nx=k1d, cfl=0.0625)
    ms, r = rate(c, 20 if k1d < 512 else 10)
    print(f"SBP N=4 K1D={k1d:4d} K={c.K:7d}: {ms:8.3f} ms/step {r:7.2f} GDOF*stages/s", flush=True)
