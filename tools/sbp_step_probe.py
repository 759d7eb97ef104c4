#!/usr/bin/env python3
"""SBP N=4 FAST step timing as production runs it (graph replay, PDL, no per-launch
timers): CUDA events over `steps` LSRK45 steps on the handle's stream, reported per RK
stage and as a fraction of the FP64 peak on the SURVEY §8(d) flop count.  Library variant
via SWEDG_LIB_VARIANT, whole-step launch via SWEDG_SBP_CHAIN (0/1).

    python tools/sbp_step_probe.py [K1D ...]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_02516_b200 import capi  # noqa: E402

FLOP = 55 * 666 + 33 * 15 + 7 * 37  # SURVEY §8(d) SBP N=4 volume+surface accounting
peak = capi.probe_fp64_peak(0, 3)
tag = os.path.basename(os.environ.get("SWEDG_LIB_VARIANT", "default")) + " chain=" + os.environ.get("SWEDG_SBP_CHAIN", "1")
for k1d in [int(x) for x in sys.argv[1:]] or [128, 256]:
    c = capi.Case("dambreak", scheme=capi.SCHEME_SBP, N=4, nx=k1d, cfl=0.0625)
    h = c.handle(mode=capi.MODE_FAST, diagnostics=False)
    st = torch.cuda.Stream()
    h.set_stream(st.cuda_stream)
    h.set_state(c.u0())
    h.step(c.dt, 3)
    steps = max(10, 60 * (128 // k1d) ** 2)
    best = None
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        h.step(c.dt, steps, sync=False)
        e1.record(st)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / (5 * steps)
        best = ms if best is None else min(best, ms)
    tf = FLOP * c.K / (best * 1e-3) / 1e12
    print(f"[{tag}] K1D={k1d} K={c.K}: {best * 1e3:.1f} us per stage, {tf:.2f} TFLOP/s = {tf / peak:.3f} of {peak:.1f}",
          flush=True)
    h.close()
    c.close()
