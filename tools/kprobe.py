#!/usr/bin/env python3
"""Per-kernel CUDA-event timing of the FAST stage kernels (volume / interface class)
for the modal N=4 smooth-wave case (C4 workload at a given K1D) and the SBP N=4 dam
break (C3), against the FP64 roofline (SURVEY §8(d) flop counts).

    python tools/kprobe.py [modal K1D] [sbp K1D] [steps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_02516_b200 import capi  # noqa: E402

MODAL_N = int(os.environ.get("KPROBE_N", "4"))
# projection + volume + volume lift per element (SURVEY §8(d) accounting)
MODAL_FLOP = {3: 3996 + 17356 + 6 * 10 * 16, 4: 48340}[MODAL_N]
SBP_FLOP = 55 * 666 + 33 * 15 + 7 * 37       # SURVEY §8(d) SBP N=4


def run(case, flop, steps, label):
    h = case.handle()
    st = torch.cuda.Stream()
    h.set_stream(st.cuda_stream)
    h.set_state(case.u0())
    h.step(case.dt, 3)
    h.enable_timers(True)
    h.read_timers()
    h.step(case.dt, steps)
    ms, n = h.read_timers()
    h.enable_timers(False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    h.step(case.dt, steps, sync=False)
    e1.record(st)
    torch.cuda.synchronize()
    h.check()
    v = ms[0] / max(n[0], 1)
    tf = flop * case.K / (v * 1e-3) / 1e12
    print(f"{label} K={case.K}: class0 {v * 1e3:.1f} us x{n[0]} ({tf:.2f} TFLOP/s = {tf / PEAK:.3f}), "
          f"class1 {ms[1] / max(n[1], 1) * 1e3:.1f} us x{n[1]}, step {e0.elapsed_time(e1) / steps:.3f} ms", flush=True)
    h.close()


if __name__ == "__main__":
    mk = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    sk = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    PEAK = capi.probe_fp64_peak(0, 3)
    print(f"fp64 peak {PEAK:.2f} TFLOP/s", flush=True)
    if mk > 0:
        run(capi.Case("smooth", N=MODAL_N, nx=mk, warp=0.1, seed=23), MODAL_FLOP, steps, f"modal N={MODAL_N} K1D={mk}")
    if sk > 0:
        run(capi.Case("dambreak", scheme=capi.SCHEME_SBP, N=4, nx=sk, cfl=0.0625), SBP_FLOP, steps, f"sbp N=4 K1D={sk}")
