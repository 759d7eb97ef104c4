"""Element partitioning and the per-stage halo exchange (multi-rank path).

The RHS is element-local except the exterior face trace u~+ (solver.hpp:263-264),
so the mesh shards by elements with ONE exchange per RK stage: the face traces
of boundary elements, between swedg_stage_volume (which writes the owned traces)
and swedg_stage_surface (which reads owned + halo traces).

Partition = y-strips of the structured periodic mesh (native setup
`Case(..., strips=P, strip=r)`): rank r owns quad rows [r*ny, (r+1)*ny) of a
global nx x (ny*P) mesh; its halo slots are
    below  K + [0, 2nx)      <- rank r-1's last owned row  (elements K-2nx .. K-1)
    above  K + 2nx + [0,2nx) <- rank r+1's first owned row (elements 0 .. 2nx-1)
(periodic wrap in y).  Traces of whole elements ([3][nf] blocks) are shipped:
2nx*45 doubles per neighbour per stage (737 KB at nx=1024) — latency-bound on
NVLink, hidden behind the ms-scale volume kernel.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class StripHalo:
    P: int
    rank: int
    nx: int
    K: int  # owned elements

    @property
    def row(self) -> int:
        return 2 * self.nx

    @property
    def prev(self) -> int:
        return (self.rank - 1) % self.P

    @property
    def next(self) -> int:
        return (self.rank + 1) % self.P

    # (begin, end) element ranges in the [K + n_halo] trace buffer
    @property
    def send_to_next(self):  # my last row -> next rank's below-halo
        return (self.K - self.row, self.K)

    @property
    def send_to_prev(self):  # my first row -> prev rank's above-halo
        return (0, self.row)

    @property
    def recv_from_prev(self):  # below-halo
        return (self.K, self.K + self.row)

    @property
    def recv_from_next(self):  # above-halo
        return (self.K + self.row, self.K + 2 * self.row)


def exchange(trace, plan: StripHalo, group=None) -> None:
    """Fill the halo slots of `trace` ([K + 4nx][3][nf] torch tensor, CPU or CUDA)
    from the neighbouring ranks with point-to-point messages (NCCL or gloo).
    Issue order is identical on every rank, so for P = 2 (both neighbours are the
    same rank) the two messages each way still pair up in order."""
    import torch.distributed as dist

    if plan.P == 1:
        return
    if trace.is_cuda and dist.get_backend(group) == "gloo":  # gloo P2P needs host tensors
        host = trace.cpu()
        exchange(host, plan, group)
        c0, c1 = plan.recv_from_prev
        d0, d1 = plan.recv_from_next
        trace[c0:c1].copy_(host[c0:c1])
        trace[d0:d1].copy_(host[d0:d1])
        return
    a0, a1 = plan.send_to_next
    b0, b1 = plan.send_to_prev
    c0, c1 = plan.recv_from_prev
    d0, d1 = plan.recv_from_next
    ops = [
        dist.P2POp(dist.isend, trace[a0:a1].contiguous(), plan.next, group),
        dist.P2POp(dist.isend, trace[b0:b1].contiguous(), plan.prev, group),
    ]
    rb = trace[c0:c1]
    ra = trace[d0:d1]
    ops += [dist.P2POp(dist.irecv, rb, plan.prev, group), dist.P2POp(dist.irecv, ra, plan.next, group)]
    for r in dist.batch_isend_irecv(ops):
        r.wait()


def stage_overlapped(h, stage: int, dt: float, trace, plan: StripHalo, stream, comm_stream, group=None,
                     exchange_fn=None) -> None:
    """One LSRK45 stage with the halo exchange overlapped with interior volume work:
    the volume kernel runs first on the two boundary rows (the elements whose traces
    the neighbours need), the exchange of those traces starts on `comm_stream`, the
    interior volume kernel runs on `stream` meanwhile, and the surface kernel waits
    for the exchange.  `exchange_fn(trace, plan)` defaults to `exchange` (NCCL/gloo
    point-to-point)."""
    import torch

    K, row = plan.K, plan.row
    ex = exchange_fn or (lambda t, p: exchange(t, p, group))
    h.stage_volume_range(stage, dt, 0, row)            # first row  -> previous rank
    h.stage_volume_range(stage, dt, K - row, K)        # last row   -> next rank
    boundary_done = torch.cuda.Event()
    boundary_done.record(stream)
    with torch.cuda.stream(comm_stream):
        comm_stream.wait_event(boundary_done)
        ex(trace, plan)
        halos_in = torch.cuda.Event()
        halos_in.record(comm_stream)
    h.stage_volume_range(stage, dt, row, K - row)      # interior, concurrent with the exchange
    stream.wait_event(halos_in)
    h.stage_surface(stage, dt)


def state_tensor(handle):
    """Zero-copy torch view [K][3][Np] of a handle's device-resident state."""
    import torch

    u_ptr, _ = handle.state_device_ptrs()
    s = handle.sizes
    return torch.as_tensor(_CudaArray(u_ptr, (s.K, 3, handle.nstate)), device="cuda")


class HostStepper:
    """Host-state LSRK45 steps of one rank (the multi-rank counterpart of
    swedg_step_lsrk45_host): every step copies the rank's state in from a pinned
    host buffer and its result back out, and the copies overlap the work:
    the two boundary rows arrive first, the stage-0 volume kernel runs chunk by chunk
    as the rest lands (the halo exchange starts after the boundary rows), and the
    last interface kernel runs chunk by chunk, each chunk's D2H starting at once.
    Stages 1..3 use stage_overlapped."""

    def __init__(self, h, plan: StripHalo, stream, comm_stream, chunks: int = 16, group=None, exchange_fn=None):
        import torch

        self.h, self.plan, self.stream, self.comm = h, plan, stream, comm_stream
        self.group, self.exchange_fn = group, exchange_fn
        K, row = plan.K, plan.row
        inner = max(1, min(chunks - 2, (K - 2 * row) // max(1, row)))
        cuts = [row + (K - 2 * row) * i // inner for i in range(inner + 1)]
        # processing order: first row, last row, then the interior from the bottom up
        self.ranges = [(0, row), (K - row, K)] + [(cuts[i], cuts[i + 1]) for i in range(inner) if cuts[i] < cuts[i + 1]]
        self.copy_in = torch.cuda.Stream(device=stream.device)
        self.copy_out = torch.cuda.Stream(device=stream.device)
        n = len(self.ranges)
        self.ev_in = [torch.cuda.Event() for _ in range(n)]
        self.ev_out = [torch.cuda.Event() for _ in range(n)]
        self.ev_done = [torch.cuda.Event() for _ in range(n)]
        self.trace = trace_tensor(h)
        self.dev = state_tensor(h)

    def _exchange(self):
        ex = self.exchange_fn or (lambda t, p: exchange(t, p, self.group))
        ex(self.trace, self.plan)

    def step(self, host_u, dt: float, nsteps: int = 1) -> None:
        """host_u: torch CPU tensor (pinned) [K][3][Np], updated in place every step."""
        import torch

        h, st, comm = self.h, self.stream, self.comm
        K, row = self.plan.K, self.plan.row
        ready = torch.cuda.Event()
        ready.record(st)
        self.copy_in.wait_event(ready)
        for n in range(nsteps):
            for i, (a, b) in enumerate(self.ranges):  # H2D, after the previous step's D2H of the chunk
                if n > 0:
                    self.copy_in.wait_event(self.ev_out[i])
                with torch.cuda.stream(self.copy_in):
                    self.dev[a:b].copy_(host_u[a:b], non_blocking=True)
                self.ev_in[i].record(self.copy_in)
            with torch.cuda.stream(st):
                for s in range(5):
                    if s in (1, 2, 3):
                        stage_overlapped(h, s, dt, self.trace, self.plan, st, comm, self.group, self.exchange_fn)
                        continue
                    # boundary rows first (stage 0: as they land), exchange on the comm stream
                    for i in (0, 1):
                        if s == 0:
                            st.wait_event(self.ev_in[i])
                        h.stage_volume_range(s, dt, *self.ranges[i])
                    boundary = torch.cuda.Event()
                    boundary.record(st)
                    with torch.cuda.stream(comm):
                        comm.wait_event(boundary)
                        self._exchange()
                        halos = torch.cuda.Event()
                        halos.record(comm)
                    for i in range(2, len(self.ranges)):
                        if s == 0:
                            st.wait_event(self.ev_in[i])
                        h.stage_volume_range(s, dt, *self.ranges[i])
                    st.wait_event(halos)
                    if s == 0:
                        h.stage_surface(s, dt)
                        continue
                    # last stage: interface kernel by chunk (the range ending at K last), D2H right after
                    order = sorted(range(len(self.ranges)), key=lambda i: self.ranges[i][1] == K)
                    for i in order:
                        a, b = self.ranges[i]
                        h.stage_surface_range(s, dt, a, b)
                        self.ev_done[i].record(st)
                        self.copy_out.wait_event(self.ev_done[i])
                        with torch.cuda.stream(self.copy_out):
                            host_u[a:b].copy_(self.dev[a:b], non_blocking=True)
                        self.ev_out[i].record(self.copy_out)
        for e in self.ev_out:
            st.wait_event(e)


def copy_halos_local(traces, plans) -> None:
    """Single-process stand-in for `exchange` over P logical partitions (device copies)."""
    P = len(plans)
    for r, pl in enumerate(plans):
        prv, nxt = plans[pl.prev], plans[pl.next]
        c0, c1 = pl.recv_from_prev
        a0, a1 = prv.send_to_next
        traces[r][c0:c1].copy_(traces[pl.prev][a0:a1])
        d0, d1 = pl.recv_from_next
        b0, b1 = nxt.send_to_prev
        traces[r][d0:d1].copy_(traces[pl.next][b0:b1])
    assert P >= 1


class _CudaArray:
    def __init__(self, ptr: int, shape, typestr="<f8"):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def trace_tensor(handle):
    """Zero-copy torch view [K + n_halo][3][nf] of a handle's device face-trace buffer."""
    import torch

    ptr, K, H = handle.trace_info()
    nf = handle.sizes.nf
    return torch.as_tensor(_CudaArray(ptr, (K + H, 3, nf)), device="cuda")
