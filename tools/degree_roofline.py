#!/usr/bin/env python3
"""Roofline fractions of the FAST stage kernels for every degree N = 1..4 on the C4
generator (smooth wave + lake bathymetry, curved, K1D given): per-kernel CUDA-event
timers; volume kernel against the in-run FP64 peak (SURVEY §8(d) flop accounting,
bench.flops_bytes_per_element), interface kernel against MEASURED_PEAKS.json HBM.

    python tools/degree_roofline.py [K1D]"""
import json
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench  # noqa: E402
from paper_2005_02516_b200 import capi  # noqa: E402

k1d = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
peak = capi.probe_fp64_peak(0, 5)
try:
    hbm = float(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"])
except Exception:  # the driver writes MEASURED_PEAKS.json; B200_PROFILING.md's measured copy rate
    hbm = 6452.8
for N in (1, 2, 3, 4):
    c = capi.Case("smooth", N=N, nx=k1d, warp=0.1, seed=23)
    h = c.handle(mode=capi.MODE_FAST, diagnostics=False)
    st = torch.cuda.Stream()
    h.set_stream(st.cuda_stream)
    h.set_state(c.u0())
    h.step(c.dt, 3)
    h.enable_timers(True)
    h.read_timers()
    h.step(c.dt, 5)
    ms, n = h.read_timers()
    fb = bench.flops_bytes_per_element(N)
    v, s = ms[0] / n[0], ms[1] / n[1]
    tf = fb["vol_flops"] * c.K / (v * 1e-3) / 1e12
    gbs = fb["surf_bytes"] * c.K / (s * 1e-3) / 1e9
    dofs = c.K * c.Np * 3 * 5 / ((ms[0] + ms[1]) / 5 * 1e-3) / 1e9
    print(json.dumps({"N": N, "K": c.K, "volume_ms": round(v, 4), "volume_tflops": round(tf, 3),
                      "volume_frac": round(tf / peak, 4), "interface_ms": round(s, 4), "interface_gbs": round(gbs, 1),
                      "interface_frac": round(gbs / hbm, 4), "gdof_stages_s": round(dofs, 3),
                      "vol_flops_per_elem": fb["vol_flops"], "surf_bytes_per_elem": fb["surf_bytes"],
                      "fp64_peak": round(peak, 2), "hbm_peak": hbm}), flush=True)
    h.close()
    c.close()
