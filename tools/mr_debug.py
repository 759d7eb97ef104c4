"""Step-by-step probe of the multi-rank paths with hard timeouts (debugging aid)."""
import faulthandler
import sys
import time

import numpy as np

sys.path.insert(0, ".")
faulthandler.dump_traceback_later(60, exit=True)
from paper_2005_02516_b200 import capi  # noqa: E402
from paper_2005_02516_b200.partition import LocalExchange  # noqa: E402

which = sys.argv[1]
N, P = 4, int(sys.argv[2]) if len(sys.argv) > 2 else 1
g = capi.Case("smooth", N=N, nx=6, ny=7, warp=0.1)
hg = g.handle()
hg.set_state(g.u0())
hg.step(1e-3, 3)
ug = hg.get_state()[0]
print("global done", flush=True)
cases = [capi.Case("smooth", N=N, nx=6, ny=7, warp=0.1, strips=P, strip=r, scaling="strong") for r in range(P)]
hs = [c.handle() for c in cases]
for h, c in zip(hs, cases):
    h.set_state(c.u0())
print("handles", [h.halo_ranges() for h in hs], flush=True)
if which == "stage":
    for s in range(5):
        print("stage", s, flush=True)
        hs[0].stage_volume(s, 1e-3)
        hs[0].halo_pack()
        hs[0].check()
        print(" vol+pack ok", flush=True)
        hs[0].stage_surface(s, 1e-3)
        hs[0].check()
elif which == "nocopy":
    hs[0].set_exchange(lambda st, a, b, c: print("cb", st, flush=True))
    hs[0].step(1e-3, 1, sync=True)
    print("step ok", flush=True)
elif which == "local":
    LocalExchange(hs, [c.halo_desc() for c in cases], cases[0].nf).step(1e-3, 3)
    u = np.concatenate([h.get_state()[0] for h in hs])
    print("local bitwise:", np.array_equal(u, ug), flush=True)
elif which == "nccl":
    comm = capi.nccl_comm_init(1, capi.nccl_unique_id(), 0, 0)
    print("comm", comm, flush=True)
    hs[0].set_nccl_comm(comm)
    hs[0].step(1e-3, 1)
    print("1 step ok", flush=True)
    hs[0].step(1e-3, 2)
    print("graph ok", np.array_equal(hs[0].get_state()[0], ug), flush=True)
elif which == "nccl2":  # two communicators one after the other
    for NN in (3, 4):
        c = capi.Case("smooth", N=NN, nx=6, ny=7, warp=0.1, strips=1, strip=0, scaling="strong")
        h = c.handle()
        h.set_state(c.u0())
        comm = capi.nccl_comm_init(1, capi.nccl_unique_id(), 0, 0)
        h.set_nccl_comm(comm)
        h.step(1e-3, 4)
        print("N", NN, "ok", flush=True)
        h.close()
        capi.nccl_comm_destroy(comm)
print("done", flush=True)
