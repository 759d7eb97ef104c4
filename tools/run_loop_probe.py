#!/usr/bin/env python3
"""Where the device run loop's time goes (swedg_run, run.hpp:226-262) on the small configs:
CUDA events on the handle's stream around (a) the run loop alone, (b) the same number of
steps alone, (c) the same number of invariant samples alone.

    python tools/run_loop_probe.py"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_02516_b200 import capi  # noqa: E402

CONFIGS = [("C1", "vortex", 3, capi.SCHEME_HYBRIDIZED, 16, 0.0, 0.125, 0.5),
           ("C2", "lake", 3, capi.SCHEME_HYBRIDIZED, 16, 0.1, 0.125, 0.5),
           ("C3", "dambreak", 4, capi.SCHEME_SBP, 128, 0.0, 0.0625, 0.05)]


def timed(st, fn, reset, reps=3):
    best = None
    for _ in range(reps):
        reset()  # every repetition from the initial state (C3 loses positivity at t ~ 0.07)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.time()
        e0.record(st)
        fn()
        e1.record(st)
        e1.synchronize()
        r = (e0.elapsed_time(e1), (time.time() - w0) * 1e3)
        best = r if best is None or r[0] < best[0] else best
    return best


for name, prob, N, scheme, n, warp, cfl, tf in CONFIGS:
    c = capi.Case(prob, N=N, nx=n, warp=warp, cfl=cfl, scheme=scheme)
    h = c.handle(mode=capi.MODE_FAST)
    st = torch.cuda.Stream()
    h.set_stream(st.cuda_stream)
    u0 = c.u0()
    h.set_state(u0)
    _, nsteps = h.run(c.dt, tf)
    ns = nsteps + 1

    def reset():
        h.set_state(u0, None, 0.0)

    a = timed(st, lambda: h.run(c.dt, tf), reset)
    b = timed(st, lambda: h.step(c.dt, nsteps, sync=False), reset)
    cc = timed(st, lambda: [h.sample_invariants(i) for i in range(ns)], reset)
    h.check()
    print(f"{name} K={c.K} steps={nsteps}: run loop {a[0]:.2f} ms (wall {a[1]:.2f}); steps alone {b[0]:.2f} ms "
          f"({b[0] / nsteps * 1e3:.1f} us/step); {ns} samples alone {cc[0]:.2f} ms ({cc[0] / ns * 1e3:.1f} us/sample)",
          flush=True)
    h.close()
    c.close()
