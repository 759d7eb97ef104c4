#!/usr/bin/env python3
"""Device-resident C4 steps over a long window (power-capped regime): ms/step and the
SM clock / power sampled by nvidia-smi during the window."""
import os
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_02516_b200 import capi  # noqa: E402

nsteps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
case = capi.Case("smooth", N=4, nx=1024, warp=0.1, seed=23)
h = case.handle()
st = torch.cuda.Stream()
h.set_stream(st.cuda_stream)
h.set_state(case.u0())
h.step(case.dt, 5)
torch.cuda.synchronize()
samples = []
stop = threading.Event()


def sampler():
    while not stop.is_set():
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True).stdout.strip().split(",")
        try:
            samples.append((float(out[0]), float(out[1])))
        except Exception:
            pass
        time.sleep(0.2)


th = threading.Thread(target=sampler)
th.start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
h.step(case.dt, nsteps, sync=False)
e1.record(st)
torch.cuda.synchronize()
stop.set()
th.join()
h.check()
clk = sorted(s[0] for s in samples)
pw = sorted(s[1] for s in samples)
print(f"{os.environ.get('SWEDG_LIB_VARIANT', 'default')}: {e0.elapsed_time(e1) / nsteps:.3f} ms/step, "
      f"SM MHz median {clk[len(clk) // 2] if clk else 0:.0f}, power median {pw[len(pw) // 2] if pw else 0:.0f} W", flush=True)
