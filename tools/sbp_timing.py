#!/usr/bin/env python3
"""SBP N=4 kernel timing (C3 dam break and a larger K) with per-kernel CUDA-event timers:
volume/interface kernel vs the FP64 roofline (~37.4 K flop per element)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_02516_b200 import capi  # noqa: E402

FLOP = 55 * 666 + 33 * 15 + 7 * 37  # SURVEY §8(d) SBP N=4 volume+surface accounting
peak = capi.probe_fp64_peak(0, 3)
for k1d in (128, 256):
    c = capi.Case("dambreak", scheme=capi.SCHEME_SBP, N=4, nx=k1d, cfl=0.0625)
    h = c.handle()
    st = torch.cuda.Stream()
    h.set_stream(st.cuda_stream)
    h.set_state(c.u0())
    h.step(c.dt, 3)
    h.enable_timers(True)
    h.read_timers()
    h.step(c.dt, 10)
    ms, n = h.read_timers()
    vol = ms[0] / n[0]
    tf = FLOP * c.K / (vol * 1e-3) / 1e12
    print(f"K1D={k1d} K={c.K}: rhs kernel {vol * 1e3:.1f} us ({tf:.2f} TFLOP/s = {tf / peak:.3f} of {peak:.1f}), "
          f"update {ms[1] / n[1] * 1e3:.1f} us, step {(ms[0] + ms[1]) / 10:.3f} ms", flush=True)
    h.close()
