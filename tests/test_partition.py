"""Multi-rank path: y-strip partitions with a per-stage halo exchange of cut-face traces.

CPU tests (this container):
  * the strip setup (weak and strong scaling) equals the global mesh bitwise, and its
    halo map points every cut face at the right neighbour trace;
  * real multi-process runs (torch.distributed gloo, world size 2 and 3): every rank
    steps its strip with the C oracle, exchanging only the packed cut-face traces in
    the wire format each stage; the gathered state after 2 LSRK45 steps equals the
    single-process global run bit for bit.
GPU tests: the native multi-rank schedule (swedg_capi.cu run_step_halo) with logical
partitions on one device (one host thread per rank, exchange callback with device
copies), with a one-rank NCCL communicator (self exchange across the periodic cut,
inside the captured step graph), and the stage-level API — all bitwise equal to the
unpartitioned steps.
"""
import os
import socket

import numpy as np
import pytest
import torch

from oracle_py import Oracle, case_dict
from paper_2005_02516_b200 import capi
from paper_2005_02516_b200.partition import LocalExchange, exchange_messages, message_offsets, pack_faces

NX, NY, N = 6, 3, 3  # weak: 6 x 3 quads per rank; strong: the 6 x 7 mesh cut in P strips
NY_STRONG = 7
LSRK_A = (0.0, -0.41789047449985195, -1.192151694642677, -1.6977846924715279, -1.5141834442571558)
LSRK_B = (0.14965902199922912, 0.37921031299962726, 0.8229550293869817, 0.6994504559491221, 0.15305724796815198)


def rows(scaling, P, r):
    """Global quad rows [j0, j1) owned by rank r."""
    if scaling == "weak":
        return r * NY, (r + 1) * NY
    return NY_STRONG * r // P, NY_STRONG * (r + 1) // P


def case(scaling, P, r, N=N, **kw):
    ny = NY if scaling == "weak" else NY_STRONG
    return capi.Case("smooth", N=N, nx=NX, ny=ny, warp=0.1, strips=P, strip=r, scaling=scaling, threads=1, **kw)


def stride(c):
    """Field stride of a halo pseudo-element: modal face traces [3][nf], SBP states [3][nq]."""
    return c.nq if c.scheme == capi.SCHEME_SBP else c.nf


def owned_slice(scaling, P, r):
    j0, j1 = rows(scaling, P, r)
    return slice(2 * NX * j0, 2 * NX * j1)


def halo_source(halos, P, r, slot_face):
    """(source rank, sender's element, sender's face) of halo face `slot_face` = 3 q + position
    of rank r, following the message pairing rule (k-th send a -> b = b's k-th receive from a)."""
    h = halos[r]
    base = 0
    for m, (n, src) in enumerate(zip(h["recv_count"], h["recv_peer"])):
        if slot_face < base + 3 * ((int(n) + 2) // 3):
            j = slot_face - base
            k = sum(1 for mm in range(m) if int(h["recv_peer"][mm]) == int(src))
            hs = halos[int(src)]
            sent = [i for i, d in enumerate(hs["send_peer"]) if int(d) == r][k]
            first = int(np.sum(hs["send_count"][:sent]))
            return int(src), int(hs["send_elem"][first + j]), int(hs["send_face"][first + j])
        base += 3 * ((int(n) + 2) // 3)
    raise AssertionError("halo slot outside the receive messages")


@pytest.mark.parametrize("scheme", [capi.SCHEME_HYBRIDIZED, capi.SCHEME_SBP])
@pytest.mark.parametrize("scaling,P", [("weak", 2), ("weak", 3), ("strong", 1), ("strong", 2), ("strong", 3)])
def test_strip_setup_matches_global_mesh(scaling, P, scheme):
    g = case(scaling, P, -1, scheme=scheme)
    Kg = g.K
    assert g.n_halo == 0
    gnbr = g.iarray("nbr").reshape(Kg, 3)
    gperm = g.iarray("perm").reshape(Kg, -1)
    strips = [case(scaling, P, r, scheme=scheme) for r in range(P)]
    halos = [s.halo_desc() for s in strips]
    dt = min(s.dt for s in strips)
    assert dt == g.dt  # owned minimum edges: the global dt exactly
    npf = g.npf
    for r, s in enumerate(strips):
        K = s.K
        sl = owned_slice(scaling, P, r)
        assert K == sl.stop - sl.start
        assert s.n_halo == 2 * ((NX + 2) // 3)  # nx cut faces per side, 3 per halo slot
        ns = s.nstate
        extra = [("J_vol", s.nq)] if scheme == capi.SCHEME_SBP else [("Mh_inv", s.Np * s.Np)]
        for name, per in [("gf", 4 * (s.nq + s.nf)), ("sJ", s.nf), ("nx", s.nf), ("u0", 3 * ns), ("b", ns)] + extra:
            np.testing.assert_array_equal(s.array(name).reshape(K, per), g.array(name).reshape(Kg, per)[sl],
                                          err_msg=name)
        lnbr = s.iarray("nbr").reshape(K, 3)
        lperm = s.iarray("perm").reshape(K, -1)
        for k in range(K):
            for f in range(3):
                n = int(lnbr[k, f])
                gk = sl.start + k
                if n < K:
                    assert n + sl.start == gnbr[gk, f]
                    np.testing.assert_array_equal(lperm[k, f * npf:(f + 1) * npf], gperm[gk, f * npf:(f + 1) * npf])
                    continue
                pos = lperm[k, f * npf] // npf
                src, e, fe = halo_source(halos, P, r, 3 * (n - K) + pos)
                assert owned_slice(scaling, P, src).start + e == gnbr[gk, f], (r, k, f)
                for sn in range(npf):  # node order: global perm = (neighbour face) npf + node
                    assert lperm[k, f * npf + sn] // npf == pos
                    assert gperm[gk, f * npf + sn] == fe * npf + lperm[k, f * npf + sn] % npf


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, P, scaling, port, dt, nsteps, q, scheme=capi.SCHEME_HYBRIDIZED):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=P)
    try:
        s = case(scaling, P, rank, scheme=scheme)
        c = case_dict(s)
        halo = s.halo_desc()
        orc = Oracle(c)
        K, nq, nf, npf, nh = s.K, s.nq, s.nf, s.npf, s.nq + s.nf
        blk = stride(s)
        nrecv = sum(ln for _, ln in message_offsets(halo["recv_count"], blk))
        assert nrecv == s.n_halo * 3 * blk
        u = np.array(c["u"], copy=True)
        res = np.zeros_like(u)
        for _ in range(nsteps):
            for st in range(5):
                recv = torch.zeros(nrecv, dtype=torch.float64)
                if scheme == capi.SCHEME_SBP:  # the neighbours' states at the cut faces' nodes
                    send = torch.from_numpy(pack_faces(u, halo, npf, s.iarray("face_index")))
                    exchange_messages(send, recv, halo, blk)
                    du, err, _ = orc.rhs(np.concatenate([u, recv.numpy().reshape(s.n_halo, 3, nq)]))
                else:
                    proj, err, _ = orc.entropy_projection(u)
                    assert err == 0
                    send = torch.from_numpy(pack_faces(proj[:, :, nq:], halo, npf))
                    exchange_messages(send, recv, halo, nf)  # cut-face traces only, wire format
                    proj_all = np.zeros((K + s.n_halo, 3, nh))
                    proj_all[:K] = proj
                    proj_all[K:, :, nq:] = recv.numpy().reshape(s.n_halo, 3, nf)
                    du, err, _ = orc.rhs_from_proj(proj_all)
                assert err == 0
                res = LSRK_A[st] * res + dt * du  # step_lsrk45 (solver.hpp:479-480)
                u = u + LSRK_B[st] * res
        q.put((rank, u, int(send.numel())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("scaling,P,scheme", [("strong", 2, 0), ("strong", 3, 0), ("weak", 2, 0), ("strong", 2, 1),
                                              ("strong", 3, 1)])
def test_gloo_partitioned_steps_equal_global_bitwise(scaling, P, scheme):
    """World size P over gloo: 2 LSRK45 steps with per-stage cut-face exchanges (modal: face
    traces; SBP: face-node states); the gathered state equals the single-process global run
    (C oracle = the reference's arithmetic) bitwise."""
    import torch.multiprocessing as mp

    dt, nsteps = 1e-3, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, P, scaling, port, dt, nsteps, q, scheme)) for r in range(P)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(P):
        r, u, nsend = q.get(timeout=600)
        got[r] = (u, nsend)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = case(scaling, P, -1, scheme=scheme)
    gc = case_dict(g)
    ug, _, err = Oracle(gc).step_lsrk45(gc["u"], np.zeros_like(gc["u"]), dt, nsteps)
    assert err == 0
    for r in range(P):
        np.testing.assert_array_equal(got[r][0], ug[owned_slice(scaling, P, r)])
        # only the cut faces travel: 2 messages of nx faces, 3 faces per pseudo-element
        assert got[r][1] == 2 * ((NX + 2) // 3) * 3 * stride(g)


# ---------------------------------------------------------------------------- GPU
def _global_steps(g, dt, nsteps, N, mode=capi.MODE_FAST):
    hg = g.handle(mode=mode)
    hg.set_state(g.u0())
    hg.step(dt, nsteps)
    ug, _, tg = hg.get_state()
    hg.close()
    return ug, tg


@pytest.mark.gpu
@pytest.mark.parametrize("scheme,N,mode", [(0, 3, "fast"), (0, 4, "fast"), (0, 4, "parity"), (1, 4, "fast"),
                                           (1, 3, "fast"), (1, 4, "parity")])
@pytest.mark.parametrize("scaling,P", [("strong", 1), ("strong", 2), ("strong", 3), ("weak", 2)])
def test_native_multirank_step_logical_partitions(scaling, P, scheme, N, mode):
    """swedg_step_lsrk45 on P strip handles (one host thread each, exchange callback pushing
    the packed cut faces into the peers' halo slots by device copies) == the global steps,
    bitwise (modal: boundary-first volume ranges, comm stream, interior overlap; SBP:
    interior RHS during the exchange, then the cut-face elements; FAST pair kernels and
    PARITY kernels)."""
    dt, nsteps = 1e-3, 3
    m = capi.MODE_FAST if mode == "fast" else capi.MODE_PARITY
    g = case(scaling, P, -1, N=N, scheme=scheme)
    ug, tg = _global_steps(g, dt, nsteps, N, m)
    cases = [case(scaling, P, r, N=N, scheme=scheme) for r in range(P)]
    hs = [c.handle(mode=m) for c in cases]
    for h, c in zip(hs, cases):
        h.set_state(c.u0())
    LocalExchange(hs, [c.halo_desc() for c in cases], stride(cases[0])).step(dt, nsteps)
    for r, h in enumerate(hs):
        u, _, t = h.get_state()
        np.testing.assert_array_equal(u, ug[owned_slice(scaling, P, r)])
        assert t == tg


@pytest.mark.gpu
@pytest.mark.parametrize("P,nchunks", [(1, 3), (2, 4), (3, 16)])
def test_multirank_host_state_steps_equal_global(P, nchunks):
    """swedg_step_lsrk45_host on strip handles (H2D by element ranges, the ranges owning
    sent faces first; stage-0 volume kernels wait per range; the last interface kernel by
    ranges, each range's D2H right after it) == the global device-resident steps, bitwise;
    the host buffers hold every step's result."""
    dt, nsteps = 1e-3, 3
    g = case("strong", P, -1, N=4)
    ug, tg = _global_steps(g, dt, nsteps, 4)
    cases = [case("strong", P, r, N=4) for r in range(P)]
    hs = [c.handle(mode=capi.MODE_FAST) for c in cases]
    us = [np.ascontiguousarray(c.u0()) for c in cases]
    for h, u in zip(hs, us):
        h.set_state(u)
    LocalExchange(hs, [c.halo_desc() for c in cases], stride(cases[0])).step_host(us, dt, nsteps, nchunks)
    for r, (h, u) in enumerate(zip(hs, us)):
        np.testing.assert_array_equal(u, ug[owned_slice("strong", P, r)])
        ud, _, t = h.get_state()
        np.testing.assert_array_equal(ud, u)
        assert t == tg


@pytest.mark.gpu
def test_nccl_self_exchange_single_rank_graph():
    """One rank whose halos are its own periodic cut (strong, P = 1) with a one-rank NCCL
    communicator: ncclSend/ncclRecv to itself inside the captured step graph (the
    production multi-GPU code path on one device) == the unpartitioned steps, bitwise."""
    dt = 1e-3
    for scheme, N in ((0, 3), (0, 4), (1, 4)):
        g = case("strong", 1, -1, N=N, scheme=scheme)
        ug, tg = _global_steps(g, dt, 4, N)
        c = case("strong", 1, 0, N=N, scheme=scheme)
        h = c.handle(mode=capi.MODE_FAST)
        comm = capi.nccl_comm_init(1, capi.nccl_unique_id(), 0, 0)
        try:
            h.set_nccl_comm(comm)
            h.set_state(c.u0())
            h.step(dt, 3)  # graph capture + replay
            h.set_graphs(False)
            h.step(dt, 1)  # individual launches
            u, _, t = h.get_state()
        finally:
            h.close()  # the handle's captured graph holds NCCL work: it goes before the comm
            capi.nccl_comm_destroy(comm)
        np.testing.assert_array_equal(u, ug)
        assert t == tg


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 3])
def test_stage_level_pack_and_device_copies(P):
    """The stage-level API (volume ranges, swedg_halo_pack, caller-moved messages,
    interface kernel) with logical partitions == the global steps, bitwise; also checks
    the stage ids when volume ranges are issued out of order (interior first)."""
    from paper_2005_02516_b200.partition import _view

    dt, nsteps = 1e-3, 2
    g = case("strong", P, -1, N=4)
    ug, _ = _global_steps(g, dt, nsteps, 4)
    cases = [case("strong", P, r, N=4) for r in range(P)]
    hs = [c.handle(mode=capi.MODE_FAST) for c in cases]
    halos = [c.halo_desc() for c in cases]
    nf = cases[0].nf
    for h, c in zip(hs, cases):
        h.set_state(c.u0())
    bufs = [h.halo_buffers() for h in hs]
    for _ in range(nsteps):
        for s in range(5):
            for h in hs:
                bnd, inner = h.halo_ranges()
                for a, b in inner + bnd:  # any order within a stage
                    h.stage_volume_range(s, dt, a, b)
                h.halo_pack()
            torch.cuda.synchronize()
            for q in range(P):  # receive message m of q from its k-th send partner
                seen = {}
                for (off, ln), src in zip(message_offsets(halos[q]["recv_count"], nf), halos[q]["recv_peer"]):
                    src = int(src)
                    k = seen.get(src, 0)
                    seen[src] = k + 1
                    sends = [i for i, d in enumerate(halos[src]["send_peer"]) if int(d) == q]
                    soff, sln = message_offsets(halos[src]["send_count"], nf)[sends[k]]
                    _view(bufs[q][2] + 8 * off, (ln,)).copy_(_view(bufs[src][0] + 8 * soff, (sln,)))
            torch.cuda.synchronize()
            for h in hs:
                h.stage_surface(s, dt)
    for r, h in enumerate(hs):
        h.check()
        u, _, _ = h.get_state()
        np.testing.assert_array_equal(u, ug[owned_slice("strong", P, r)])


@pytest.mark.gpu
def test_multirank_handle_without_transport_fails_loudly():
    c = case("strong", 2, 0, N=4)
    h = c.handle(mode=capi.MODE_FAST)
    h.set_state(c.u0())
    with pytest.raises(capi.InvalidArgument):
        h.step(1e-3, 1)


@pytest.mark.gpu
@pytest.mark.parametrize("scheme", [capi.SCHEME_HYBRIDIZED, capi.SCHEME_SBP])
def test_multirank_run_loop_invariants_equal_global(scheme):
    """run() on P = 3 logical partitions: the device time loop per rank (graph-free steps
    with the exchange callback, invariants sampled per rank), raw exact accumulators merged
    — the invariant series and the final state equal the single-GPU run() bit for bit."""
    P, N = 3, 4
    g = case("strong", P, -1, N=N, scheme=scheme)
    dt = g.dt
    hg = g.handle(mode=capi.MODE_FAST)
    hg.set_state(g.u0())
    sg, ng = hg.run(dt, 12 * dt, sample_every=4)
    ug, _, _ = hg.get_state()
    cases = [case("strong", P, r, N=N, scheme=scheme) for r in range(P)]
    hs = [c.handle(mode=capi.MODE_FAST) for c in cases]
    for h, c in zip(hs, cases):
        h.set_state(c.u0())
    s, n = LocalExchange(hs, [c.halo_desc() for c in cases], stride(cases[0])).run(dt, 12 * dt, 4)
    assert n == ng and len(s) == len(sg) == 4
    np.testing.assert_array_equal(s, sg)
    for r, h in enumerate(hs):
        np.testing.assert_array_equal(h.get_state()[0], ug[owned_slice("strong", P, r)])


# ---------------------------------------------------------------- peer-memory transport
@pytest.mark.gpu
@pytest.mark.timeout(600)
@pytest.mark.parametrize("scheme,N,mode", [(0, 3, "fast"), (0, 4, "fast"), (0, 4, "parity"), (1, 4, "fast"),
                                           (1, 4, "parity")])
def test_p2p_self_exchange_single_rank(scheme, N, mode):
    """Peer-memory transport on one rank whose halos are its own periodic cut (strong,
    P = 1): the pack kernel stores into its own halo slots and the stream flag protocol
    runs against itself.  3 graph-replayed steps (flag waits/writes are graph nodes) + 1
    individual step == the global steps, bitwise."""
    from paper_2005_02516_b200.partition import attach_p2p_local

    dt = 1e-3
    m = capi.MODE_FAST if mode == "fast" else capi.MODE_PARITY
    g = case("strong", 1, -1, N=N, scheme=scheme)
    ug, tg = _global_steps(g, dt, 4, N, m)
    c = case("strong", 1, 0, N=N, scheme=scheme)
    h = c.handle(mode=m)
    h.set_state(c.u0())
    attach_p2p_local([h])
    h.step(dt, 3)
    h.set_graphs(False)
    h.step(dt, 1)
    u, _, t = h.get_state()
    np.testing.assert_array_equal(u, ug)
    assert t == tg


def _p2p_case(scaling, P, r, scheme, job):
    if job == "hostwave":
        return capi.Case("smooth", N=4, nx=6, ny=16 * P, warp=0.1, strips=P, strip=r, scaling="strong", threads=1,
                         scheme=scheme)
    return case(scaling, P, r, N=4, scheme=scheme)


def _p2p_rank_main(rank, P, scaling, scheme, mode, job, dt, port, q):
    """One rank per process (the production layout; here every process on device 0): halo
    slots and flags of the peers mapped through CUDA IPC, descriptors over gloo."""
    import torch.distributed as dist

    from paper_2005_02516_b200.partition import attach_p2p

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=P)
    try:
        torch.cuda.set_device(0)
        c = _p2p_case(scaling, P, rank, scheme, job)
        h = c.handle(mode=capi.MODE_FAST if mode == "fast" else capi.MODE_PARITY)
        u0 = np.ascontiguousarray(c.u0())
        h.set_state(u0)
        attach_p2p(h, rank, P)
        dist.barrier()
        out = {}
        if job == "steps":
            h.step(1e-3, 3)  # captured step graph, replayed
            h.set_graphs(False)
            h.step(1e-3, 1)  # individual launches
            out["u"] = h.get_state()[0]
        elif job == "host":
            h.step_host(u0, 1e-3, 3, 4)  # range-chunked host-state steps
            out["u"] = u0
        elif job == "hostwave":  # a strip tall enough for the host-state wavefront
            l0 = h.launches
            h.step_host(u0, 1e-3, 3, 4)
            out["u"] = u0
            out["wavefront"] = h.launches - l0 == wave_launches(5 * 3, 4)
        else:  # run loop with invariant sampling: raw exact accumulators for the merge
            series, n = h.run(dt, 8 * dt, 4)  # the global mesh's dt
            out["raw"] = h.read_invariants_raw(len(series))
            out["n"] = (len(series), n)
            out["u"] = h.get_state()[0]
        dist.barrier()  # no rank unmaps its peers' buffers before their last stores
        h.close()
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.timeout(300)
@pytest.mark.parametrize("scaling,P,scheme,mode,job", [
    ("strong", 2, 0, "fast", "steps"), ("strong", 3, 0, "fast", "steps"), ("weak", 2, 0, "fast", "steps"),
    ("weak", 2, 1, "fast", "steps"), ("weak", 3, 0, "parity", "steps"),
    ("strong", 3, 0, "parity", "steps"), ("strong", 2, 1, "fast", "steps"), ("strong", 3, 1, "fast", "steps"),
    ("strong", 3, 1, "parity", "steps"), ("strong", 3, 0, "fast", "host"), ("strong", 3, 0, "fast", "hostwave"),
    ("strong", 3, 0, "fast", "run"), ("strong", 3, 1, "fast", "run")])
def test_p2p_processes_equal_global_bitwise(scaling, P, scheme, mode, job):
    """Peer-memory transport with one rank per process (CUDA IPC): each rank's pack kernel
    stores its cut faces straight into the peers' halo slots, the ranks' streams order the
    stages through flags in each other's memory (no host sync).  Graph-replayed and
    individual steps, host-state steps and the run loop (raw invariants merged) all equal
    the single-rank results bit for bit."""
    import torch.multiprocessing as mp

    m = capi.MODE_FAST if mode == "fast" else capi.MODE_PARITY
    g = _p2p_case(scaling, P, -1, scheme, job)
    hg = g.handle(mode=m)
    hg.set_state(g.u0())
    if job == "run":
        sg, ng = hg.run(g.dt, 8 * g.dt, sample_every=4)
    else:
        hg.step(1e-3, 3 if job.startswith("host") else 4)
    ug = hg.get_state()[0]
    hg.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_p2p_rank_main, args=(r, P, scaling, scheme, mode, job, g.dt, port, q))
             for r in range(P)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=600) for _ in range(P))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for r in range(P):
        if job == "hostwave":
            j0, j1 = 16 * P * r // P, 16 * P * (r + 1) // P
            np.testing.assert_array_equal(got[r]["u"], ug[12 * j0:12 * j1])
            assert got[r]["wavefront"]
        else:
            np.testing.assert_array_equal(got[r]["u"], ug[owned_slice(scaling, P, r)])
    if job == "run":
        n = got[0]["n"][0]
        assert got[0]["n"] == (len(sg), ng)
        np.testing.assert_array_equal(capi.diag_from_raw([got[r]["raw"] for r in range(P)], n), sg)


@pytest.mark.gpu
def test_p2p_attach_errors_are_loud():
    """swedg_set_p2p refuses a rank that did not export its descriptor, descriptors in the
    wrong rank order and halo maps that disagree; a detached handle steps again only with
    a transport."""
    c0, c1 = case("strong", 2, 0, N=4), case("strong", 2, 1, N=4)
    h0, h1 = c0.handle(mode=capi.MODE_FAST), c1.handle(mode=capi.MODE_FAST)
    b1 = h1.p2p_export(1)
    with pytest.raises(capi.InvalidArgument, match="export"):
        h0.set_p2p(0, [b1, b1])  # rank 0 never exported
    b0 = h0.p2p_export(0)
    with pytest.raises(capi.InvalidArgument, match="not a swedg_p2p_export of rank 0"):
        h0.set_p2p(0, [b1, b0])
    g = case("strong", 3, 1, N=4).handle(mode=capi.MODE_FAST)  # a 3-strip rank: other message sizes
    with pytest.raises(capi.InvalidArgument, match="disagree"):
        h0.set_p2p(0, [b0, g.p2p_export(1)])
    h0.set_p2p(0, [b0, b1])
    h0.set_p2p(0, None)
    h0.set_state(c0.u0())
    with pytest.raises(capi.InvalidArgument):
        h0.step(1e-3, 1)


@pytest.mark.gpu
@pytest.mark.parametrize("P,C", [(1, 4), (2, 4), (3, 8)])
def test_multirank_host_state_wavefront_equal_global(P, C):
    """swedg_step_lsrk45_host on strip handles tall enough for the wavefront schedule (each
    rank's first and last rows in the ring's first chunks): the per-stage exchange is
    enqueued after the boundary chunks' volume kernels inside the wavefront, the boundary
    interface kernels wait for it.  Bitwise the global device-resident steps; the launch
    count shows the wavefront ran: per tick one segmented launch of the volume pieces and one
    of the interface pieces (at most 4 per launch), 1 pack per stage."""
    ny, dt, nsteps = 16 * P, 1e-3, 3

    def mk(r):
        return capi.Case("smooth", N=4, nx=6, ny=ny, warp=0.1, strips=P, strip=r, scaling="strong", threads=1)

    g = mk(-1)
    ug, tg = _global_steps(g, dt, nsteps, 4)
    cases = [mk(r) for r in range(P)]
    hs = [c.handle(mode=capi.MODE_FAST) for c in cases]
    us = [np.ascontiguousarray(c.u0()) for c in cases]
    for h, u in zip(hs, us):
        h.set_state(u)
    l0 = [h.launches for h in hs]
    LocalExchange(hs, [c.halo_desc() for c in cases], cases[0].nf).step_host(us, dt, nsteps, C)
    row = 2 * 6
    for r, (h, u) in enumerate(zip(hs, us)):
        j0, j1 = ny * r // P, ny * (r + 1) // P
        np.testing.assert_array_equal(u, ug[row * j0:row * j1])
        assert h.launches - l0[r] == wave_launches(5 * nsteps, C)
        assert h.get_state()[2] == tg


def wave_launches(G, C):
    """Launches of the host-state wavefront over G stages with C chunks (N = 4 FAST):
    volume pieces (g, p) go out at tick 6 g + p and interface pieces at 6 g + p + 3, merged
    per tick in launches of <= 4 pieces; one pack per stage."""
    ticks = {}
    for g in range(G):
        for p in range(C):
            ticks[6 * g + p] = ticks.get(6 * g + p, 0) + 1
    return 2 * sum((n + 3) // 4 for n in ticks.values()) + G
