"""Multi-rank path: y-strip partitions with a per-stage halo exchange of face traces.

CPU tests (this container): the strip setup equals the global mesh bitwise, and
a real multi-process run (torch.distributed gloo, world size 2 and 3) that
computes each rank's RHS with the C oracle from its owned elements plus halo
traces received over gloo reproduces the single-process global RHS bit for bit.
GPU test: P logical partitions on one device (halo moved by device copies,
never kernels waiting on each other) equal the unpartitioned run bitwise.
"""
import os
import socket

import numpy as np
import pytest
import torch

from oracle_py import Oracle, case_dict
from paper_2005_02516_b200 import capi
from paper_2005_02516_b200.partition import StripHalo, copy_halos_local, exchange

NX, NY, N = 6, 3, 3  # per-strip quads: 6 x 3 -> 36 owned elements per rank


def owned_slice(r):
    return slice(r * NY * 2 * NX, (r + 1) * NY * 2 * NX)


@pytest.mark.parametrize("P", [2, 3])
def test_strip_setup_matches_global_mesh(P):
    g = capi.Case("smooth", N=N, nx=NX, ny=NY, warp=0.1, strips=P, strip=-1, threads=1)
    Kg = g.K
    assert Kg == 2 * NX * NY * P and g.n_halo == 0
    gnbr = g.iarray("nbr").reshape(Kg, 3)
    for r in range(P):
        s = capi.Case("smooth", N=N, nx=NX, ny=NY, warp=0.1, strips=P, strip=r, threads=1)
        K = s.K
        assert K == 2 * NX * NY and s.n_halo == 4 * NX
        sl = owned_slice(r)
        for name, per in [("gf", 4 * (s.nq + s.nf)), ("Mh_inv", s.Np * s.Np), ("sJ", s.nf), ("nx", s.nf),
                          ("u0", 3 * s.Np), ("b", s.Np)]:
            np.testing.assert_array_equal(s.array(name).reshape(K, per), g.array(name).reshape(Kg, per)[sl],
                                          err_msg=name)
        np.testing.assert_array_equal(s.iarray("perm").reshape(K, -1), g.iarray("perm").reshape(Kg, -1)[sl])
        # neighbour ids: owned -> global id, halo slot -> the neighbour rank's row
        plan = StripHalo(P, r, NX, K)
        off = sl.start
        lnbr = s.iarray("nbr").reshape(K, 3)
        row = 2 * NX
        for k in range(K):
            for f in range(3):
                n = int(lnbr[k, f])
                if n < K:
                    gid = n + off
                elif n < K + row:  # below halo <- prev rank's last row
                    gid = owned_slice(plan.prev).stop - row + (n - K)
                else:  # above halo <- next rank's first row
                    gid = owned_slice(plan.next).start + (n - K - row)
                assert gid == gnbr[off + k, f], (r, k, f)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, P, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=P)
    try:
        s = capi.Case("smooth", N=N, nx=NX, ny=NY, warp=0.1, strips=P, strip=rank, threads=1)
        c = case_dict(s)
        orc = Oracle(c)
        proj, err, _ = orc.entropy_projection(c["u"])
        assert err == 0
        K, nq, nf = s.K, s.nq, s.nf
        trace = torch.zeros((K + s.n_halo, 3, nf), dtype=torch.float64)
        trace[:K] = torch.from_numpy(proj[:, :, nq:])
        exchange(trace, StripHalo(P, rank, NX, K))
        proj_all = np.zeros((K + s.n_halo, 3, nq + nf))
        proj_all[:K] = proj
        proj_all[K:, :, nq:] = trace[K:].numpy()
        du, err, _ = orc.rhs_from_proj(proj_all)
        assert err == 0
        q.put((rank, du))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P", [2, 3])
def test_gloo_partitioned_rhs_equals_global_bitwise(P):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, P, port, q)) for r in range(P)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(P))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = capi.Case("smooth", N=N, nx=NX, ny=NY, warp=0.1, strips=P, strip=-1, threads=1)
    gc = case_dict(g)
    du_g, err, _ = Oracle(gc).rhs(gc["u"])
    assert err == 0
    for r in range(P):
        np.testing.assert_array_equal(got[r], du_g[owned_slice(r)])


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 3])
def test_logical_partitions_on_one_gpu_equal_global(P):
    from paper_2005_02516_b200.partition import trace_tensor

    g = capi.Case("smooth", N=4, nx=NX, ny=NY, warp=0.1, strips=P, strip=-1, threads=1)
    hg = g.handle(mode=capi.MODE_FAST)
    hg.set_state(g.u0())
    dt = 1e-3
    hg.step(dt, 2)
    ug, _, _ = hg.get_state()
    cases = [capi.Case("smooth", N=4, nx=NX, ny=NY, warp=0.1, strips=P, strip=r, threads=1) for r in range(P)]
    hs = [c.handle(mode=capi.MODE_FAST) for c in cases]
    for h, c in zip(hs, cases):
        h.set_state(c.u0())
    plans = [StripHalo(P, r, NX, c.K) for r, c in enumerate(cases)]
    traces = [trace_tensor(h) for h in hs]
    for _ in range(2):
        for s in range(5):
            for h in hs:
                h.stage_volume(s, dt)
            torch.cuda.synchronize()
            copy_halos_local(traces, plans)
            torch.cuda.synchronize()
            for h in hs:
                h.stage_surface(s, dt)
    for h in hs:
        h.check()
    for r, h in enumerate(hs):
        u, _, t = h.get_state()
        np.testing.assert_array_equal(u, ug[owned_slice(r)])
        assert t == 2 * dt


@pytest.mark.gpu
@pytest.mark.parametrize("N", [3, 4])
@pytest.mark.parametrize("P", [2, 3])
def test_boundary_first_volume_ranges_equal_global(P, N):
    """The overlapped schedule (partition.stage_overlapped): boundary rows' volume kernel,
    halo exchange, interior volume kernel, surface kernel — with logical partitions on
    one GPU — bit-for-bit the unpartitioned steps (N=4 and N=3 pair kernels)."""
    from paper_2005_02516_b200.partition import trace_tensor

    g = capi.Case("smooth", N=N, nx=NX, ny=NY, warp=0.1, strips=P, strip=-1, threads=1)
    hg = g.handle(mode=capi.MODE_FAST)
    hg.set_state(g.u0())
    dt = 1e-3
    hg.step(dt, 2)
    ug, _, _ = hg.get_state()
    cases = [capi.Case("smooth", N=N, nx=NX, ny=NY, warp=0.1, strips=P, strip=r, threads=1) for r in range(P)]
    hs = [c.handle(mode=capi.MODE_FAST) for c in cases]
    for h, c in zip(hs, cases):
        h.set_state(c.u0())
    plans = [StripHalo(P, r, NX, c.K) for r, c in enumerate(cases)]
    traces = [trace_tensor(h) for h in hs]
    for _ in range(2):
        for s in range(5):
            for h, pl in zip(hs, plans):
                h.stage_volume_range(s, dt, 0, pl.row)
                h.stage_volume_range(s, dt, pl.K - pl.row, pl.K)
            torch.cuda.synchronize()
            copy_halos_local(traces, plans)
            for h, pl in zip(hs, plans):
                h.stage_volume_range(s, dt, pl.row, pl.K - pl.row)
            torch.cuda.synchronize()
            for h in hs:
                h.stage_surface(s, dt)
    for h in hs:
        h.check()
    for r, h in enumerate(hs):
        u, _, t = h.get_state()
        np.testing.assert_array_equal(u, ug[owned_slice(r)])


@pytest.mark.gpu
def test_stage_overlapped_single_rank_equals_step():
    """partition.stage_overlapped on one rank (no neighbours: the exchange is empty) with
    separate compute and comm streams == swedg_step_lsrk45, bitwise."""
    from paper_2005_02516_b200.partition import stage_overlapped, trace_tensor

    c = capi.Case("smooth", N=4, nx=NX, ny=NY, warp=0.1, threads=1)
    dt = 1e-3
    h1 = c.handle(mode=capi.MODE_FAST)
    h1.set_state(c.u0())
    h1.step(dt, 2)
    u1, _, _ = h1.get_state()
    h2 = c.handle(mode=capi.MODE_FAST)
    stream, comm = torch.cuda.Stream(), torch.cuda.Stream()
    h2.set_stream(stream.cuda_stream)
    h2.set_state(c.u0())
    plan = StripHalo(1, 0, NX, c.K)
    trace = trace_tensor(h2)
    with torch.cuda.stream(stream):
        for _ in range(2):
            for s in range(5):
                stage_overlapped(h2, s, dt, trace, plan, stream, comm)
    torch.cuda.synchronize()
    h2.check()
    u2, _, _ = h2.get_state()
    np.testing.assert_array_equal(u1, u2)


@pytest.mark.gpu
def test_host_stepper_single_rank_equals_step():
    """partition.HostStepper (per-rank host-state steps with chunked copies overlapping the
    stage-0 volume and last interface kernels) on one rank == swedg_step_lsrk45, bitwise,
    and the host buffer holds every step's result."""
    from paper_2005_02516_b200.partition import HostStepper

    c = capi.Case("smooth", N=4, nx=NX, ny=8, warp=0.1, threads=1)
    dt = 1e-3
    h1 = c.handle(mode=capi.MODE_FAST)
    h1.set_state(c.u0())
    h1.step(dt, 3)
    u1, _, t1 = h1.get_state()
    h2 = c.handle(mode=capi.MODE_FAST)
    stream, comm = torch.cuda.Stream(), torch.cuda.Stream()
    h2.set_stream(stream.cuda_stream)
    h2.set_state(c.u0())
    hu = torch.from_numpy(c.u0().copy()).pin_memory()
    hs = HostStepper(h2, StripHalo(1, 0, NX, c.K), stream, comm, chunks=5)
    hs.step(hu, dt, 3)
    torch.cuda.synchronize()
    h2.check()
    np.testing.assert_array_equal(hu.numpy(), u1)
    u2, _, t2 = h2.get_state()
    np.testing.assert_array_equal(u2, u1)
    assert t2 == t1
