"""Configs C3 (SBP N=4 dam break, K1D=128) and C5-size (modal N=4, K1D=2048 on one GPU):
build with the native setup, run LSRK45 steps on the device, report time per step,
throughput and invariants.  Prints JSON lines (recorded in DESIGN.md / profiles/)."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2005_02516_b200 import capi  # noqa: E402


def mass(case, u):
    # integral of h with the volume rule: sum_k sum_i w_i J_i h_i (nodal SBP) / modal via Vq
    w = case.array("volq_w")
    J = case.array("J_vol").reshape(case.K, case.nq)
    if case.scheme == capi.SCHEME_SBP:
        return float((w[None, :] * J * u[:, 0, :]).sum())
    Vq = case.array("Vq").reshape(case.Np, case.nq).T  # stored [cols][rows]
    hq = u[:, 0, :] @ Vq.T
    return float((w[None, :] * J * hq).sum())


def run(name, case, steps, mode=capi.MODE_FAST):
    h = case.handle(mode=mode)
    u0 = case.u0()
    h.set_state(u0)
    m0 = mass(case, u0)
    h.step(case.dt, 2)
    s = torch.cuda.ExternalStream(h.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    h.step(case.dt, steps, sync=False)
    e1.record(s)
    torch.cuda.synchronize()
    h.check()
    ms = e0.elapsed_time(e1) / steps
    u, _, t = h.get_state()
    m1 = mass(case, u)
    dof = case.K * case.nstate * 3
    print(json.dumps({"config": name, "K": case.K, "dof": dof, "ms_per_step": round(ms, 3),
                      "gdof_stages_per_s": round(dof * 5 / (ms * 1e-3) / 1e9, 3), "steps": steps + 2,
                      "t": t, "min_h": float(u[:, 0, :].min()) if case.scheme == 1 else None,
                      "mass_rel_drift": abs(m1 - m0) / abs(m0), "device_GB": round(h.device_bytes / 1e9, 2)}),
          flush=True)
    h.close()


if __name__ == "__main__":
    t0 = time.time()
    c3 = capi.Case("dambreak", scheme=capi.SCHEME_SBP, N=4, nx=128, cfl=0.0625)
    print(f"# C3 setup {time.time() - t0:.1f}s dt={c3.dt:.3e}", flush=True)
    run("C3 SBP N=4 dam break K1D=128", c3, 200)
    if len(sys.argv) > 1 and sys.argv[1] == "c5":
        t0 = time.time()
        c5 = capi.Case("smooth", N=4, nx=2048, warp=0.1)
        print(f"# C5 setup {time.time() - t0:.1f}s", flush=True)
        run("C5-size modal N=4 K1D=2048 (1 GPU)", c5, 5)
