"""Quick throughput probe: tile a golden periodic fixture into R disjoint copies
(each copy keeps its own periodic connectivity) and time LSRK45 steps."""
import os
import sys
import time

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))
from oracle_py import load_golden  # noqa: E402

from paper_2005_02516_b200 import capi  # noqa: E402


def tiled(c, R):
    K = int(c["K"][0])
    out = dict(c)
    per = ["gf", "sJ", "nx", "ny", "Mh_inv", "u", "b", "J_vol"]
    for k in per:
        if k in c:
            out[k] = np.concatenate([c[k]] * R, axis=0)
    nbr = c["nbr"]
    out["nbr"] = np.concatenate([np.where(nbr >= 0, nbr + r * K, -1) for r in range(R)], axis=0)
    out["perm"] = np.concatenate([c["perm"]] * R, axis=0)
    out["K"] = np.array([K * R], dtype=np.int32)
    return out


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "modal_n4_warp"
    R = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
    mode = capi.MODE_PARITY if (len(sys.argv) > 3 and sys.argv[3] == "parity") else capi.MODE_FAST
    c = tiled(load_golden(name), R)
    K = int(c["K"][0])
    t0 = time.time()
    h = capi.handle_from_case(c, mode=mode)
    h.set_state(c["u"])
    print(f"{name} K={K} setup {time.time() - t0:.1f}s dev_bytes={h.device_bytes / 1e9:.2f} GB", flush=True)
    s = torch.cuda.ExternalStream(h.stream)
    dt = 1e-5
    h.step(dt, 2)
    torch.cuda.synchronize()
    nsteps = 5
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    h.step(dt, nsteps, sync=False)
    e1.record(s)
    torch.cuda.synchronize()
    h.check()
    ms = e0.elapsed_time(e1)
    nloc = c["u"].shape[2]
    dof = K * 3 * nloc
    stages = 5 * nsteps
    print(f"  {ms / stages:.3f} ms/stage  {dof * stages / (ms * 1e-3) / 1e9:.3f} GDOF*stages/s", flush=True)


if __name__ == "__main__":
    main()
