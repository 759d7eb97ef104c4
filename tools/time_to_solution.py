#!/usr/bin/env python3
"""Time to solution of the small BASELINE configs (C1, C2, C3): the reference's own
build_case + run() on the host cores (oracle/_ref/swedg_refbench run, all cores and one
thread) against the device run loop run.run() (graph-replayed steps, device invariant
samples, final L2 error on the device) through the C ABI, FAST mode.  GPU times are wall
clock around run.run() after one warm run (state reset by run.run), and the device-side
share measured with CUDA events on the handle's stream.

    python tools/time_to_solution.py [--ref-threads N] > profiles/r2_time_to_solution.json"""
import argparse
import json
import os
import subprocess
import sys
import time

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2005_02516_b200 import capi, run  # noqa: E402

# (name, problem, N, scheme, K1D, warp, cfl, tfinal); C3's dam break loses positivity in the
# reference's own arithmetic at t ~ 0.070 (no limiter), so it runs to t = 0.05
CONFIGS = [("C1", "vortex", 3, "hybridized", 16, 0.0, 0.125, 0.5),
           ("C2", "lake", 3, "hybridized", 16, 0.1, 0.125, 0.5),
           ("C3", "dambreak", 4, "sbp", 128, 0.0, 0.0625, 0.05)]


def ref_run(cfg, threads):
    _, prob, N, scheme, n, warp, cfl, tf = cfg
    exe = os.path.join(REPO, "oracle", "_ref", "swedg_refbench")
    out = subprocess.run([exe, "run", prob, str(N), scheme, str(n), str(warp), str(cfl), str(tf), str(threads)],
                         capture_output=True, text=True, timeout=3600, check=True)
    return json.loads(out.stdout.strip().splitlines()[-1])


def gpu_run(cfg):
    name, prob, N, scheme, n, warp, cfl, tf = cfg
    t0 = time.time()
    c = capi.Case(prob, N=N, nx=n, warp=warp, cfl=cfl,
                  scheme=capi.SCHEME_SBP if scheme == "sbp" else capi.SCHEME_HYBRIDIZED)
    setup = time.time() - t0
    h = c.handle(mode=capi.MODE_FAST)
    st = torch.cuda.Stream()
    h.set_stream(st.cuda_stream)
    run.run(c, tfinal=tf, handle=h)  # warm: graph capture, first-touch
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t1 = time.time()
    e0.record(st)
    r = run.run(c, tfinal=tf, handle=h)
    e1.record(st)
    torch.cuda.synchronize()
    wall = time.time() - t1
    out = {"K": c.K, "steps": int(r.get("steps", 0)) if isinstance(r, dict) else None, "run_s": wall,
           "device_s": e0.elapsed_time(e1) / 1e3, "setup_s": setup}
    if isinstance(r, dict) and r.get("error"):
        out["l2_h"] = float(r["error"].get("err_h", float("nan")))
    h.close()
    c.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref-threads", type=int, default=os.cpu_count())
    a = ap.parse_args()
    rows = []
    for cfg in CONFIGS:
        g = gpu_run(cfg)
        rm = ref_run(cfg, a.ref_threads)
        r1 = ref_run(cfg, 1)
        rows.append({"config": cfg[0], "problem": cfg[1], "N": cfg[2], "scheme": cfg[3], "K1D": cfg[4],
                     "tfinal": cfg[7], "gpu": g, "reference": rm, "reference_1thread": r1,
                     "speedup_vs_reference": rm["run_s"] / g["run_s"], "speedup_vs_1thread": r1["run_s"] / g["run_s"]})
        print(json.dumps(rows[-1]), flush=True)


if __name__ == "__main__":
    main()
