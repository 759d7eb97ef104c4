"""Element partitioning and the per-stage halo exchange (multi-rank path).

The RHS is element-local except the exterior face trace u~+ (solver.hpp:263-264),
so the mesh shards by elements with ONE exchange per RK stage: the projected
traces of the cut faces (3 fields x npf nodes per face).

Partition = y-strips of the structured periodic mesh, built by the native setup
(`capi.Case(..., strips=P, strip=r, scaling="weak"|"strong")`, setup.cpp
compact_strip): rank r owns a band of quad rows; its halo is the two cuts' faces.
The exchange map (`Case.halo_desc()`, C ABI `swedg_halo_desc`) lists per message
the peer rank and the sent faces; the wire format packs three faces per [3][nf]
pseudo-element, the layout of the receiver's halo slots (no unpack step).

Transports (all drive the same native stage schedule, swedg_capi.cu run_step_halo:
boundary volume -> pack -> exchange on a comm stream || interior volume -> interface):
  * peer   `attach_p2p`: the pack kernel stores the cut-face traces straight into the
             peers' halo slots over NVLink peer memory (IPC-mapped), ordered by stream-
             written/-waited flags in the ranks' memory, inside the captured step graph
             (swedg_set_p2p) — the one-node production path (bench.py --gpus N).
  * NCCL   `attach_nccl`: a library-owned communicator (swedg_nccl_comm_init; the
             unique id travels over torch.distributed), ncclSend/ncclRecv inside the
             captured step graph (bench.py --transport nccl).
  * gloo   `attach_gloo`: a host-staged exchange callback (functional check of the
             multi-rank orchestration with several ranks sharing one GPU).
  * local  `LocalExchange`: P handles in one process on one GPU, one host thread per
             rank, device copies between their buffers ordered by CUDA events.
"""
from __future__ import annotations

import threading

import numpy as np


def wire_slots(n: int) -> int:
    """Pseudo-elements ([3][nf] blocks) of a message of n faces."""
    return (n + 2) // 3


def message_offsets(counts, nf: int):
    """(offset, length) in doubles of each message in a buffer of back-to-back messages."""
    out, off = [], 0
    for n in counts:
        ln = wire_slots(int(n)) * 3 * nf
        out.append((off, ln))
        off += ln
    return out


# ---------------------------------------------------------------------------
# wire format on host arrays (CPU reference of the pack kernel, halo.cuh)
def pack_faces(blocks, halo: dict, npf: int, face_index=None) -> np.ndarray:
    """Cut faces -> the send buffer (messages back to back, wire format).  Modal: blocks =
    face traces [K][3][nf]; SBP: blocks = states [K][3][nq] and face_index maps a face
    slot to its volume node (the pseudo-element keeps the state layout)."""
    blk = blocks.shape[2]
    node = (lambda x: x) if face_index is None else (lambda x: int(face_index[x]))
    offs = message_offsets(halo["send_count"], blk)
    buf = np.zeros(sum(ln for _, ln in offs))
    i = 0
    for (off, _), n in zip(offs, halo["send_count"]):
        for j in range(int(n)):
            e, f = int(halo["send_elem"][i]), int(halo["send_face"][i])
            i += 1
            base = off + (j // 3) * 3 * blk
            for c in range(3):
                for s in range(npf):
                    buf[base + c * blk + node((j % 3) * npf + s)] = blocks[e, c, node(f * npf + s)]
    return buf


# ---------------------------------------------------------------------------
# torch.distributed transports
def exchange_messages(send, recv, halo: dict, nf: int, group=None) -> None:
    """Point-to-point exchange of the wire-format messages (flat torch tensors, CPU for
    gloo, CUDA for NCCL).  Messages between the same two ranks pair up in issue order."""
    import torch.distributed as dist

    ops = []
    for (off, ln), peer in zip(message_offsets(halo["send_count"], nf), halo["send_peer"]):
        ops.append(dist.P2POp(dist.isend, send[off:off + ln].contiguous(), int(peer), group))
    for (off, ln), peer in zip(message_offsets(halo["recv_count"], nf), halo["recv_peer"]):
        ops.append(dist.P2POp(dist.irecv, recv[off:off + ln], int(peer), group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()


def attach_nccl(h, halo: dict, world: int, rank: int, device: int, group=None) -> int:
    """Give handle h a library-owned NCCL communicator over the ranks of the default
    torch.distributed group (the unique id is broadcast from rank 0).  Returns the comm."""
    import torch
    import torch.distributed as dist

    from . import capi

    uid = capi.nccl_unique_id() if rank == 0 else bytes(128)
    backend = dist.get_backend(group)
    t = torch.tensor(list(uid), dtype=torch.uint8, device="cuda" if backend == "nccl" else "cpu")
    dist.broadcast(t, src=0, group=group)
    comm = capi.nccl_comm_init(world, bytes(t.cpu().tolist()), rank, device)
    h.set_nccl_comm(comm)
    return comm


def attach_p2p(h, rank: int, world: int, group=None) -> None:
    """Peer-memory transport for handle h (ranks of one node): every rank's descriptor
    (swedg_p2p_export: IPC handles of its halo slots and flags) gathered over
    torch.distributed, then swedg_set_p2p.  The exchange itself never touches the host."""
    import torch.distributed as dist

    blob = h.p2p_export(rank)
    blobs = [None] * world
    dist.all_gather_object(blobs, blob, group=group)
    h.set_p2p(rank, blobs)


def attach_p2p_local(handles) -> None:
    """Peer-memory transport between P handles of this process (logical partitions, rank =
    position in the list); they exchange through each other's buffers directly."""
    blobs = [h.p2p_export(r) for r, h in enumerate(handles)]
    for r, h in enumerate(handles):
        h.set_p2p(r, blobs)


def attach_gloo(h, halo: dict, nf: int, group=None) -> None:
    """Host-staged exchange over gloo as the handle's transport callback (blocking:
    the stream is synchronised before the send buffer is read).  A functional path for
    several ranks on one device, not a performance path.  nf: field stride of a
    pseudo-element (modal: nf; SBP: nq)."""
    import torch

    send_ptr, ns, _, nr = h.halo_buffers()
    send_dev = _view(send_ptr, (ns,))

    def xfn(stage, send, recv, stream):
        st = torch.cuda.ExternalStream(stream)
        st.synchronize()
        host_send = send_dev.cpu()
        host_recv = torch.zeros(nr, dtype=torch.float64)
        exchange_messages(host_send, host_recv, halo, nf, group)
        with torch.cuda.stream(st):
            _view(recv, (nr,)).copy_(host_recv, non_blocking=False)

    h.set_exchange(xfn)


class LocalExchange:
    """P logical partitions on one device, each stepped by its own host thread through
    the native multi-rank schedule; the exchange callback of rank r pushes its messages
    into the peers' halo slots with device copies.  Ordering is by CUDA events only (no
    kernel waits on another rank's kernel): a rank's copy into a peer starts after the
    peer entered the stage's exchange (its previous interface kernel is done), and a
    rank's interface kernel starts after every copy into its slots."""

    def __init__(self, handles, halos, nf: int):
        """nf: field stride of a pseudo-element (modal: nf; SBP: nq)."""
        import torch

        self.h, self.halos, self.nf, self.P = handles, halos, nf, len(handles)
        self.bufs = [h.halo_buffers() for h in handles]
        self.recv = [b[2] for b in self.bufs]  # this stage's halo slots (SBP: the stage's input buffer)
        self.barrier = threading.Barrier(self.P)
        self.ready = [torch.cuda.Event() for _ in range(self.P)]
        self.copied = [torch.cuda.Event() for _ in range(self.P)]
        # message pairing: the k-th send r -> q matches q's k-th receive from r
        self.routes = []  # per rank: [(send offset, dest rank, dest offset, length)]
        recv_slots = []
        for q in range(self.P):
            per_src = {}
            for (off, ln), src in zip(message_offsets(halos[q]["recv_count"], nf), halos[q]["recv_peer"]):
                per_src.setdefault(int(src), []).append((off, ln))
            recv_slots.append(per_src)
        for r in range(self.P):
            used, rt = {}, []
            for (off, ln), dst in zip(message_offsets(halos[r]["send_count"], nf), halos[r]["send_peer"]):
                dst = int(dst)
                k = used.get(dst, 0)
                used[dst] = k + 1
                doff, dln = recv_slots[dst][r][k]
                assert dln == ln, "message sizes disagree between ranks"
                rt.append((off, dst, doff, ln))
            self.routes.append(rt)
        for r, h in enumerate(handles):
            h.set_exchange(self._fn(r))

    def _fn(self, r):
        import torch

        def xfn(stage, send, recv, stream):
            st = torch.cuda.ExternalStream(stream)
            self.recv[r] = recv
            self.ready[r].record(st)
            self.barrier.wait()
            for off, dst, doff, ln in self.routes[r]:
                st.wait_event(self.ready[dst])
                src = _view(self.bufs[r][0] + 8 * off, (ln,))
                dstv = _view(self.recv[dst] + 8 * doff, (ln,))
                with torch.cuda.stream(st):
                    dstv.copy_(src, non_blocking=True)
            self.copied[r].record(st)
            self.barrier.wait()
            for q in range(self.P):
                if any(d == r for _, d, _, _ in self.routes[q]):
                    st.wait_event(self.copied[q])

        return xfn

    def _threads(self, fn):
        errs, out = [], [None] * self.P

        def body(r):
            try:
                out[r] = fn(self.h[r])
            except Exception as e:  # noqa: BLE001 - re-raised below
                errs.append(e)
                self.barrier.abort()

        ts = [threading.Thread(target=body, args=(r,)) for r in range(self.P)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        if errs:
            raise errs[0]
        return out

    def step(self, dt: float, nsteps: int) -> None:
        self._threads(lambda h: h.step(dt, nsteps, sync=True))

    def step_host(self, states, dt: float, nsteps: int, nchunks: int = 0) -> None:
        """swedg_step_lsrk45_host on every rank: states[r] (host, C-contiguous float64,
        updated in place) round-trips through host memory every step."""
        hs = list(self.h)
        self._threads(lambda h: h.step_host(states[hs.index(h)], dt, nsteps, nchunks))

    def run(self, dt: float, tfinal: float, sample_every: int = 0):
        """run() (run.hpp:226-262) on every rank: the device time loop with invariant
        sampling; the ranks' exact raw invariant records are merged (swedg_diag_from_raw),
        so the series equals the single-GPU run's bit for bit.  Returns (series, steps)."""
        from . import capi

        res = self._threads(lambda h: h.run(dt, tfinal, sample_every))
        n = len(res[0][0])
        raws = [h.read_invariants_raw(n) for h in self.h]
        return capi.diag_from_raw(raws, n), res[0][1]


def merge_invariants(h, n: int, group=None):
    """Multi-process counterpart of LocalExchange.run's merge: every rank's raw invariant
    records of its last run() (n samples) gathered over torch.distributed and merged
    exactly; returns the global series [n][6] on every rank."""
    import torch.distributed as dist

    from . import capi

    raw = h.read_invariants_raw(n)
    allraw = [None] * dist.get_world_size(group)
    dist.all_gather_object(allraw, raw, group=group)
    return capi.diag_from_raw(allraw, n)


class _CudaArray:
    def __init__(self, ptr: int, shape, typestr="<f8"):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def _view(ptr: int, shape):
    import torch

    return torch.as_tensor(_CudaArray(ptr, shape), device="cuda")


def state_tensor(handle):
    """Zero-copy torch view [K][3][Np] of a handle's device-resident state."""
    u_ptr, _ = handle.state_device_ptrs()
    return _view(u_ptr, (handle.sizes.K, 3, handle.nstate))


def trace_tensor(handle):
    """Zero-copy torch view [K + n_halo][3][nf] of a handle's device face-trace buffer."""
    ptr, K, H = handle.trace_info()
    return _view(ptr, (K + H, 3, handle.sizes.nf))
