#!/usr/bin/env python3
"""Can the FP64-bound volume kernel and the HBM-bound interface kernel share the GPU?
Two independent C4-size handles on two streams: handle A runs only volume launches,
handle B only interface launches; their concurrent wall time is compared with each
alone (build with -DSWEDG_PAIR_WARPS=12 so a volume CTA leaves registers and shared
memory for interface CTAs on the same SM)."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_02516_b200 import capi  # noqa: E402

k1d = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
reps = 5
cases = [capi.Case("smooth", N=4, nx=k1d, warp=0.1, seed=23) for _ in range(2)]
hs = [c.handle() for c in cases]
st = [torch.cuda.Stream(), torch.cuda.Stream()]
for h, s, c in zip(hs, st, cases):
    h.set_stream(s.cuda_stream)
    h.set_state(c.u0())
    h.step(c.dt, 1)
torch.cuda.synchronize()
dt = cases[0].dt
K = cases[0].K


def vol():
    for _ in range(reps):
        hs[0].stage_volume_range(1, dt, 0, K)


def srf():
    for _ in range(reps):
        hs[1].stage_surface_range(1, dt, 0, K)


def timed(fns):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for f in fns:
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3 / reps


for _ in range(2):
    tv = timed([vol])
    ts = timed([srf])
    tb = timed([vol, srf])  # launched back to back on two streams: may run concurrently
    print(f"volume alone {tv:.3f} ms, interface alone {ts:.3f} ms, sum {tv + ts:.3f}, concurrent {tb:.3f} ms", flush=True)
for h in hs:
    h.check()
