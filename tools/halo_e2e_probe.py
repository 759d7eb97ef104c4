#!/usr/bin/env python3
"""Multi-rank code path on one GPU at C4 size: a one-rank strong partition of the
K1D=1024 mesh (halos = its own periodic cut) with a one-rank NCCL communicator or the
peer-memory transport against itself — device-resident steps (captured graph with the
exchange) and host-state steps (range-chunked copies), ms per step, against the
unpartitioned handle."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2005_02516_b200 import capi  # noqa: E402

k1d = int(sys.argv[1]) if len(sys.argv) > 1 else 1024


def timed(st, fn, n):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


strip = dict(strips=1, strip=0, scaling="strong")
for label, kw, tr in (("unpartitioned", {}, None), ("1-rank strip + NCCL self exchange", strip, "nccl"),
                      ("1-rank strip + peer-memory self exchange", strip, "p2p")):
    c = capi.Case("smooth", N=4, nx=k1d, warp=0.1, seed=23, **kw)
    h = c.handle(diagnostics=False)
    comm = None
    if tr == "nccl":
        comm = capi.nccl_comm_init(1, capi.nccl_unique_id(), 0, 0)
        h.set_nccl_comm(comm)
    elif tr == "p2p":
        h.set_p2p(0, [h.p2p_export(0)])
    st = torch.cuda.Stream()
    h.set_stream(st.cuda_stream)
    u0 = c.u0()
    h.set_state(u0)
    h.step(c.dt, 3)
    dev = timed(st, lambda: h.step(c.dt, 10, sync=False), 10)
    uh = torch.empty(u0.shape, dtype=torch.float64, pin_memory=True).numpy()
    uh[...] = u0
    h.set_state(uh)
    h.step_host(uh, c.dt, 1)
    hst = timed(st, lambda: h.step_host(uh, c.dt, 10), 10)
    print(f"{label}: device {dev:.2f} ms/step, host-state {hst:.2f} ms/step", flush=True)
    h.close()
    if comm:
        capi.nccl_comm_destroy(comm)
