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
