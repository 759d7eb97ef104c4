#!/usr/bin/env python3
"""Host-state stepping probe: marginal per-step cost of swedg_step_lsrk45_host vs
chunk count, and the raw pinned H2D / D2H / duplex copy rates (C4 workload)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2005_02516_b200 import capi  # noqa: E402

k1d = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
case = capi.Case("smooth", N=4, nx=k1d, warp=0.1, seed=23)
h = case.handle()
st = torch.cuda.Stream()
h.set_stream(st.cuda_stream)
u0 = case.u0()
uh = torch.empty(u0.shape, dtype=torch.float64, pin_memory=True).numpy()
uh[...] = u0
h.set_state(uh)
h.step(case.dt, 2)
torch.cuda.synchronize()
nbytes = uh.nbytes
d = torch.empty(uh.size, dtype=torch.float64, device="cuda")
hp = torch.from_numpy(uh).view(-1)
for name, fn in (("h2d", lambda: d.copy_(hp, non_blocking=True)), ("d2h", lambda: hp.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    print(f"{name}: {3 * nbytes / (time.perf_counter() - t) / 1e9:.1f} GB/s")
# duplex: D2H of one buffer while H2D of another
d2 = torch.empty_like(d)
hp2 = torch.empty(uh.size, dtype=torch.float64, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t = time.perf_counter()
with torch.cuda.stream(s1):
    d.copy_(hp, non_blocking=True)
with torch.cuda.stream(s2):
    hp2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
print(f"duplex: {2 * nbytes / (time.perf_counter() - t) / 1e9:.1f} GB/s aggregate")
for C in (1, 4, 8, 16, 32):
    res = []
    for n in (1, 4):
        torch.cuda.synchronize()
        t = time.perf_counter()
        h.step_host(uh, case.dt, n, C)
        res.append(time.perf_counter() - t)
    print(f"chunks {C}: 1 step {res[0]*1e3:.1f} ms, 4 steps {res[1]*1e3:.1f} ms, marginal {(res[1]-res[0])/3*1e3:.1f} ms/step")
torch.cuda.synchronize()
t = time.perf_counter()
h.step(case.dt, 4)
torch.cuda.synchronize()
print(f"device-resident: {(time.perf_counter() - t) / 4 * 1e3:.1f} ms/step")
