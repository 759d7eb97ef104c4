"""ctypes binding of the C ABI (include/swedg_b200.h) — the host side of the drop-in.

This is a thin, fail-loud layer: if libswedg_b200.so is missing or no CUDA
device is present, every entry point raises; there is no CPU fallback.
The C++ adapter for reference users is include/swedg_b200.hpp; this module
serves the Python tests, bench.py and __graft_entry__.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import build as _build

SWEDG_OK = 0
SWEDG_ERR_INVALID = -1
SWEDG_ERR_POSITIVITY = -2
SWEDG_ERR_NONFINITE = -3
SWEDG_ERR_CUDA = -4
SWEDG_ERR_UNSUPPORTED = -5

SCHEME_HYBRIDIZED = 0
SCHEME_SBP = 1
PENALTY_EC = 0
PENALTY_LF = 1
MODE_FAST = 0
MODE_PARITY = 1
DIAG_INVARIANTS = 0
DIAG_L2_REF = 1
DIAG_L2_VORTEX = 2
DIAG_L2_LAKE = 3
VORTEX_PARAMS = (1.0, 1.0, 0.0, 5.0, 2.0, 0.0, 0.0)  # VortexParams defaults (diagnostics.hpp:30-38)
INVARIANT_FIELDS = ("t", "mass", "momentum_x", "momentum_y", "entropy", "min_h")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class SwedgError(RuntimeError):
    """Reference: std::runtime_error thrown by rhs()/entropy_projection() (solver.hpp:176-180,288-290)."""

    def __init__(self, code: int, msg: str, elem: int = -1, t: float = 0.0):
        super().__init__(msg)
        self.code, self.elem, self.t = code, elem, t


class PositivityError(SwedgError):
    """Nonpositive water height (swe.hpp:25-32 PositivityError, wrapped at solver.hpp:176-180)."""


class NonFiniteError(SwedgError):
    """Non-finite RHS (solver.hpp:288-290, :429-431)."""


class InvalidArgument(SwedgError, ValueError):
    """std::invalid_argument (e.g. dt <= 0, solver.hpp:468)."""


class _Desc(C.Structure):
    _fields_ = [
        ("abi_version", C.c_int), ("scheme", C.c_int), ("penalty", C.c_int), ("mode", C.c_int),
        ("N", C.c_int), ("Np", C.c_int), ("nq", C.c_int), ("nf", C.c_int), ("npf", C.c_int),
        ("K", C.c_int), ("g", C.c_double), ("device", C.c_int),
        ("Vq", _dp), ("Vf", _dp), ("Pq", _dp), ("Qr", _dp), ("Qs", _dp), ("wf", _dp),
        ("face_index", _ip), ("M_diag", _dp),
        ("gf", _dp), ("sJ", _dp), ("nx", _dp), ("ny", _dp), ("J_vol", _dp), ("Mh_inv", _dp),
        ("nbr", _ip), ("perm", _ip), ("n_halo", C.c_int),
    ]


ABI_VERSION = 5
_lib = None


class _HaloDesc(C.Structure):
    _fields_ = [("n_send_msgs", C.c_int), ("send_peer", _ip), ("send_count", _ip), ("send_elem", _ip),
                ("send_face", _ip), ("n_recv_msgs", C.c_int), ("recv_peer", _ip), ("recv_count", _ip)]


# swedg_exchange_fn: int (*)(void* user, int stage, const double* send, double* recv, void* stream)
EXCHANGE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p)


class _DiagDesc(C.Structure):
    _fields_ = [("nfine", C.c_int), ("w", _dp), ("V", _dp), ("Vr", _dp), ("Vs", _dp), ("map_coeffs", _dp),
                ("Pq", _dp)]


def lib() -> C.CDLL:
    """Load the in-tree extension (building it first if sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("SWEDG_LIB_VARIANT")  # profiling tools: an alternative in-tree build
    if not path:
        path = _build.LIB
        if _build.needs_build():
            _build.build()
    if not os.path.exists(path):
        raise RuntimeError(f"CUDA extension missing: {path} (run __graft_entry__.build())")
    L = C.CDLL(path)
    vp = C.c_void_p
    L.swedg_create.argtypes = [C.POINTER(_Desc), C.POINTER(vp)]
    L.swedg_destroy.argtypes = [vp]
    L.swedg_set_stream.argtypes = [vp, vp]
    L.swedg_get_stream.argtypes = [vp]
    L.swedg_get_stream.restype = vp
    L.swedg_set_penalty.argtypes = [vp, C.c_int]
    L.swedg_set_mode.argtypes = [vp, C.c_int]
    L.swedg_set_bathymetry.argtypes = [vp, _dp]
    L.swedg_entropy_projection.argtypes = [vp, _dp, C.c_double, _dp]
    L.swedg_rhs.argtypes = [vp, _dp, C.c_double, _dp]
    L.swedg_set_state.argtypes = [vp, _dp, _dp, C.c_double]
    L.swedg_get_state.argtypes = [vp, _dp, _dp, _dp]
    L.swedg_step_lsrk45.argtypes = [vp, C.c_double, C.c_int, C.c_int]
    L.swedg_state_device_ptr.argtypes = [vp, C.POINTER(vp), C.POINTER(vp)]
    L.swedg_rhs_device.argtypes = [vp, vp, vp, C.c_double]
    L.swedg_check.argtypes = [vp]
    L.swedg_last_error.argtypes = [vp, _ip, C.POINTER(C.c_long), _dp, C.c_char_p, C.c_size_t]
    L.swedg_create_error.restype = C.c_char_p
    L.swedg_launch_count.argtypes = [vp]
    L.swedg_launch_count.restype = C.c_longlong
    L.swedg_device_bytes.argtypes = [vp]
    L.swedg_device_bytes.restype = C.c_size_t
    L.swedg_debug_bathymetry.argtypes = [vp, _dp, _dp]
    L.swedg_enable_timers.argtypes = [vp, C.c_int]
    L.swedg_read_timers.argtypes = [vp, _dp, C.POINTER(C.c_longlong), C.c_int]
    L.swedg_probe_fp64_peak.argtypes = [C.c_int, C.c_int, _dp]
    L.swedg_set_graphs.argtypes = [vp, C.c_int]
    L.swedg_stage_volume.argtypes = [vp, C.c_int, C.c_double]
    L.swedg_stage_surface.argtypes = [vp, C.c_int, C.c_double]
    L.swedg_stage_volume_range.argtypes = [vp, C.c_int, C.c_double, C.c_int, C.c_int]
    L.swedg_stage_surface_range.argtypes = [vp, C.c_int, C.c_double, C.c_int, C.c_int]
    L.swedg_trace_device_ptr.argtypes = [vp, C.POINTER(vp), C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]
    L.swedg_set_diagnostics.argtypes = [vp, C.POINTER(_DiagDesc)]
    L.swedg_compute_invariants.argtypes = [vp, _dp, C.c_double, _dp]
    L.swedg_l2_error.argtypes = [vp, C.c_int, _dp, _dp, C.c_double, _dp]
    L.swedg_diag_raw_bytes.restype = C.c_size_t
    L.swedg_diag_raw.argtypes = [vp, C.c_int, _dp, _dp, C.c_double, vp]
    L.swedg_diag_from_raw.argtypes = [vp, C.c_int, C.c_int, _dp]
    L.swedg_sample_invariants.argtypes = [vp, C.c_int]
    L.swedg_read_invariants.argtypes = [vp, C.c_int, _dp]
    L.swedg_read_invariants_raw.argtypes = [vp, C.c_int, vp]
    L.swedg_run.argtypes = [vp, C.c_double, C.c_double, C.c_int, C.c_int, _dp, _ip, _ip]
    L.swedg_exact_sum.argtypes = [_dp, C.c_size_t, _dp]
    L.swedg_step_lsrk45_host.argtypes = [vp, _dp, C.c_double, C.c_int, C.c_int]
    L.swedg_ratio_kernels.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_double, C.c_int, C.c_int,
                                      _dp, _dp, _dp]
    L.swedg_set_halo.argtypes = [vp, C.POINTER(_HaloDesc)]
    L.swedg_set_nccl_comm.argtypes = [vp, vp]
    L.swedg_set_exchange.argtypes = [vp, EXCHANGE_FN, vp]
    L.swedg_halo_buffers.argtypes = [vp, C.POINTER(vp), C.POINTER(C.c_size_t), C.POINTER(vp), C.POINTER(C.c_size_t)]
    L.swedg_halo_pack.argtypes = [vp]
    L.swedg_halo_ranges.argtypes = [vp, _ip, C.c_int, _ip, _ip]
    L.swedg_nccl_unique_id.argtypes = [vp]
    L.swedg_nccl_comm_init.argtypes = [C.c_int, vp, C.c_int, C.c_int, C.POINTER(vp)]
    L.swedg_nccl_comm_destroy.argtypes = [vp]
    L.swedg_p2p_export.argtypes = [vp, C.c_int, vp]
    L.swedg_set_p2p.argtypes = [vp, C.c_int, C.c_int, vp]
    _lib = L
    return L


EXPORTED = [
    "swedg_create", "swedg_destroy", "swedg_set_stream", "swedg_get_stream", "swedg_set_penalty",
    "swedg_set_mode", "swedg_set_bathymetry", "swedg_entropy_projection", "swedg_rhs",
    "swedg_set_state", "swedg_get_state", "swedg_step_lsrk45", "swedg_state_device_ptr",
    "swedg_rhs_device", "swedg_check", "swedg_last_error", "swedg_create_error",
    "swedg_launch_count", "swedg_device_bytes", "swedg_abi_version", "swedg_debug_bathymetry",
    "swedg_enable_timers", "swedg_read_timers", "swedg_probe_fp64_peak",
    "swedg_stage_volume", "swedg_stage_surface", "swedg_trace_device_ptr", "swedg_set_graphs",
    "swedg_set_diagnostics", "swedg_compute_invariants", "swedg_l2_error", "swedg_diag_raw_bytes",
    "swedg_diag_raw", "swedg_diag_from_raw", "swedg_sample_invariants", "swedg_read_invariants",
    "swedg_read_invariants_raw", "swedg_run", "swedg_exact_sum", "swedg_ratio_kernels",
    "swedg_step_lsrk45_host", "swedg_stage_volume_range", "swedg_stage_surface_range",
    "swedg_set_halo", "swedg_set_nccl_comm", "swedg_set_exchange", "swedg_halo_buffers", "swedg_halo_pack",
    "swedg_halo_ranges", "swedg_nccl_unique_id", "swedg_nccl_comm_init", "swedg_nccl_comm_destroy",
    "swedg_p2p_export", "swedg_set_p2p",
]
P2P_BLOB_BYTES = 4096  # SWEDG_P2P_BLOB_BYTES


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def _p(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _pi(a):
    return None if a is None else a.ctypes.data_as(_ip)


@dataclass
class Sizes:
    N: int
    Np: int
    nq: int
    nf: int
    npf: int
    K: int

    @property
    def nh(self) -> int:
        return self.nq + self.nf


class Handle:
    """One device-resident solver instance (one rank's element block)."""

    def __init__(self, *, scheme: int, N: int, Np: int, nq: int, nf: int, npf: int, K: int,
                 g: float, Qr, Qs, wf, gf, sJ, nx, ny, nbr, perm, Vq=None, Vf=None, Pq=None,
                 Mh_inv=None, face_index=None, M_diag=None, J_vol=None,
                 penalty: int = PENALTY_LF, mode: int = MODE_FAST, device: int = 0, n_halo: int = 0):
        L = lib()
        self.sizes = Sizes(N, Np, nq, nf, npf, K)
        self.scheme = scheme
        keep = []

        def f(a):
            if a is None:
                return None
            a = _f64(a)
            keep.append(a)
            return _p(a)

        def i(a):
            if a is None:
                return None
            a = _i32(a)
            keep.append(a)
            return _pi(a)

        d = _Desc()
        d.abi_version = ABI_VERSION
        d.scheme, d.penalty, d.mode = scheme, penalty, mode
        d.N, d.Np, d.nq, d.nf, d.npf, d.K = N, Np, nq, nf, npf, K
        d.g = float(g)
        d.device = device
        d.Vq, d.Vf, d.Pq, d.Qr, d.Qs, d.wf = f(Vq), f(Vf), f(Pq), f(Qr), f(Qs), f(wf)
        d.face_index, d.M_diag = i(face_index), f(M_diag)
        d.gf, d.sJ, d.nx, d.ny, d.J_vol, d.Mh_inv = f(gf), f(sJ), f(nx), f(ny), f(J_vol), f(Mh_inv)
        d.nbr, d.perm = i(nbr), i(perm)
        d.n_halo = int(n_halo)
        h = C.c_void_p()
        rc = L.swedg_create(C.byref(d), C.byref(h))
        if rc != SWEDG_OK:
            raise _err_class(rc)(rc, "swedg_create: " + L.swedg_create_error().decode())
        self._h = h
        self._lib = L
        self.nstate = nq if scheme == SCHEME_SBP else Np

    # -- lifecycle -------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            self._lib.swedg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc == SWEDG_OK:
            return
        code = C.c_int()
        elem = C.c_long()
        t = C.c_double()
        buf = C.create_string_buffer(512)
        self._lib.swedg_last_error(self._h, C.byref(code), C.byref(elem), C.byref(t), buf, 512)
        raise _err_class(rc)(rc, buf.value.decode(), elem.value, t.value)

    # -- API ------------------------------------------------------------------
    def set_stream(self, stream_ptr: int | None):
        self._check(self._lib.swedg_set_stream(self._h, C.c_void_p(stream_ptr) if stream_ptr else None))

    @property
    def stream(self) -> int:
        return self._lib.swedg_get_stream(self._h) or 0

    def set_penalty(self, penalty: int):
        self._check(self._lib.swedg_set_penalty(self._h, penalty))

    def set_mode(self, mode: int):
        self._check(self._lib.swedg_set_mode(self._h, mode))

    def set_bathymetry(self, b):
        b = _f64(b)
        self._check(self._lib.swedg_set_bathymetry(self._h, _p(b)))

    def bathymetry_products(self):
        s = self.sizes
        if self.scheme == SCHEME_SBP:
            src = np.zeros((s.K, 2, s.nq))
            self._check(self._lib.swedg_debug_bathymetry(self._h, None, _p(src)))
            return None, src
        bs = np.zeros((s.K, s.nh))
        src = np.zeros((s.K, 2, s.nh))
        self._check(self._lib.swedg_debug_bathymetry(self._h, _p(bs), _p(src)))
        return bs, src

    def entropy_projection(self, u, t: float = 0.0) -> np.ndarray:
        s = self.sizes
        u = _f64(u)
        proj = np.zeros((s.K, 3, s.nh))
        self._check(self._lib.swedg_entropy_projection(self._h, _p(u), float(t), _p(proj)))
        return proj

    def rhs(self, u, t: float = 0.0) -> np.ndarray:
        s = self.sizes
        u = _f64(u)
        du = np.zeros((s.K, 3, self.nstate))
        self._check(self._lib.swedg_rhs(self._h, _p(u), float(t), _p(du)))
        return du

    def set_state(self, u, res=None, t: float = 0.0):
        u = _f64(u)
        r = None if res is None else _f64(res)
        self._check(self._lib.swedg_set_state(self._h, _p(u), _p(r), float(t)))

    def get_state(self, u_out=None, with_res: bool = True):
        s = self.sizes
        u = np.zeros((s.K, 3, self.nstate)) if u_out is None else u_out
        r = np.zeros_like(u) if with_res else None
        t = C.c_double()
        self._check(self._lib.swedg_get_state(self._h, _p(u), _p(r), C.byref(t)))
        return u, r, t.value

    # -- stage-level stepping (multi-rank halo exchange between the two kernels)
    def stage_volume(self, stage: int, dt: float):
        self._check(self._lib.swedg_stage_volume(self._h, int(stage), float(dt)))

    def stage_volume_range(self, stage: int, dt: float, k0: int, k1: int):
        self._check(self._lib.swedg_stage_volume_range(self._h, int(stage), float(dt), int(k0), int(k1)))

    def stage_surface_range(self, stage: int, dt: float, k0: int, k1: int):
        self._check(self._lib.swedg_stage_surface_range(self._h, int(stage), float(dt), int(k0), int(k1)))

    def stage_surface(self, stage: int, dt: float):
        self._check(self._lib.swedg_stage_surface(self._h, int(stage), float(dt)))

    def trace_info(self):
        """(device pointer, n_owned, n_halo) of the face-trace buffer [K+n_halo][3][nf]."""
        p = C.c_void_p()
        a = C.c_longlong()
        b = C.c_longlong()
        self._check(self._lib.swedg_trace_device_ptr(self._h, C.byref(p), C.byref(a), C.byref(b)))
        return p.value, a.value, b.value

    # -- multi-rank halo exchange (swedg_set_halo) -------------------------------
    def set_halo(self, halo: dict):
        """halo: send_peer, send_count, send_elem, send_face, recv_peer, recv_count (int arrays;
        Case.halo_desc())."""
        a = {k: _i32(halo[k]) for k in ("send_peer", "send_count", "send_elem", "send_face", "recv_peer",
                                        "recv_count")}
        d = _HaloDesc()
        d.n_send_msgs, d.n_recv_msgs = len(a["send_peer"]), len(a["recv_peer"])
        for k, v in a.items():
            setattr(d, k, _pi(v))
        self._halo_keep = a
        self._check(self._lib.swedg_set_halo(self._h, C.byref(d)))

    def set_nccl_comm(self, comm: int | None):
        self._check(self._lib.swedg_set_nccl_comm(self._h, C.c_void_p(comm) if comm else None))

    def p2p_export(self, rank: int) -> bytes:
        """This rank's peer-memory descriptor (swedg_p2p_export; resets its exchange flags)."""
        buf = C.create_string_buffer(P2P_BLOB_BYTES)
        self._check(self._lib.swedg_p2p_export(self._h, int(rank), buf))
        return buf.raw

    def set_p2p(self, rank: int, blobs):
        """Peer-memory transport from every rank's descriptor (a list in rank order, or
        their concatenation); None detaches."""
        if blobs is None:
            self._check(self._lib.swedg_set_p2p(self._h, int(rank), 0, None))
            return
        raw = b"".join(blobs) if isinstance(blobs, (list, tuple)) else bytes(blobs)
        n = len(raw) // P2P_BLOB_BYTES
        buf = C.create_string_buffer(raw, len(raw))
        self._check(self._lib.swedg_set_p2p(self._h, int(rank), n, buf))

    def set_exchange(self, fn):
        """fn(stage, send_ptr, recv_ptr, stream_ptr) -> None, called at enqueue time on the
        host; it must enqueue on `stream_ptr` what fills recv (None detaches)."""
        if fn is None:
            self._xfn = None
            self._check(self._lib.swedg_set_exchange(self._h, EXCHANGE_FN(), None))
            return

        def tramp(user, stage, send, recv, stream):
            try:
                fn(stage, send, recv, stream)
                return 0
            except Exception:  # noqa: BLE001 - reported as a failed exchange
                import traceback

                traceback.print_exc()
                return 1

        self._xfn = EXCHANGE_FN(tramp)
        self._check(self._lib.swedg_set_exchange(self._h, self._xfn, None))

    def halo_buffers(self):
        """(send_ptr, n_send_doubles, recv_ptr, n_recv_doubles) device buffers."""
        sp, rp = C.c_void_p(), C.c_void_p()
        ns, nr = C.c_size_t(), C.c_size_t()
        self._check(self._lib.swedg_halo_buffers(self._h, C.byref(sp), C.byref(ns), C.byref(rp), C.byref(nr)))
        return sp.value, ns.value, rp.value, nr.value

    def halo_pack(self):
        self._check(self._lib.swedg_halo_pack(self._h))

    def halo_ranges(self):
        """(boundary ranges, interior ranges) of the multi-rank volume schedule."""
        nb, ni = C.c_int(), C.c_int()
        self._check(self._lib.swedg_halo_ranges(self._h, None, 0, C.byref(nb), C.byref(ni)))
        buf = np.zeros(2 * (nb.value + ni.value), dtype=np.int32)
        self._check(self._lib.swedg_halo_ranges(self._h, _pi(buf), nb.value + ni.value, None, None))
        r = [tuple(int(x) for x in buf[2 * i:2 * i + 2]) for i in range(nb.value + ni.value)]
        return r[:nb.value], r[nb.value:]

    def enable_timers(self, on: bool = True):
        self._check(self._lib.swedg_enable_timers(self._h, 1 if on else 0))

    def read_timers(self):
        ms = np.zeros(2)
        n = (C.c_longlong * 2)()
        self._check(self._lib.swedg_read_timers(self._h, _p(ms), n, 2))
        return ms, [int(n[0]), int(n[1])]

    def step(self, dt: float, nsteps: int = 1, sync: bool = True):
        self._check(self._lib.swedg_step_lsrk45(self._h, float(dt), int(nsteps), 1 if sync else 0))

    def step_host(self, u, dt: float, nsteps: int = 1, nchunks: int = 0):
        """nsteps LSRK45 steps on the host state u ([K][3][Np] float64, C-contiguous, updated
        in place; pinned memory recommended): every step round-trips through u."""
        if not (isinstance(u, np.ndarray) and u.dtype == np.float64 and u.flags.c_contiguous):
            raise ValueError("u must be a C-contiguous float64 array (updated in place)")
        self._check(self._lib.swedg_step_lsrk45_host(self._h, _p(u), float(dt), int(nsteps), int(nchunks)))

    def set_graphs(self, on: bool):
        self._check(self._lib.swedg_set_graphs(self._h, 1 if on else 0))

    def check(self):
        self._check(self._lib.swedg_check(self._h))

    def state_device_ptrs(self):
        u = C.c_void_p()
        r = C.c_void_p()
        self._check(self._lib.swedg_state_device_ptr(self._h, C.byref(u), C.byref(r)))
        return u.value, r.value

    def rhs_device(self, u_ptr: int, du_ptr: int, t: float = 0.0):
        self._check(self._lib.swedg_rhs_device(self._h, C.c_void_p(u_ptr), C.c_void_p(du_ptr), float(t)))

    # -- diagnostics (diagnostics.hpp:142-267, run.hpp:226-262) -----------------
    def set_diagnostics(self, *, w, V, Vr, Vs, map_coeffs, Pq=None):
        """FineQuad arrays (V/Vr/Vs as [Np][nfine] = column-major nfine x Np) and the
        per-element mapping coefficients [K][2][Np]; Pq for SBP (project_nodal)."""
        keep = [_f64(a) for a in (w, V, Vr, Vs, map_coeffs)] + ([_f64(Pq)] if Pq is not None else [])
        d = _DiagDesc()
        d.nfine = int(keep[0].shape[0])
        d.w, d.V, d.Vr, d.Vs, d.map_coeffs = (_p(a) for a in keep[:5])
        d.Pq = _p(keep[5]) if Pq is not None else None
        self._check(self._lib.swedg_set_diagnostics(self._h, C.byref(d)))

    def compute_invariants(self, u=None, t: float = 0.0) -> dict:
        """Invariants of u (None = the resident state at the handle's time)."""
        out = np.zeros(6)
        ua = None if u is None else _f64(u)
        self._check(self._lib.swedg_compute_invariants(self._h, _p(ua), float(t), _p(out)))
        return dict(zip(INVARIANT_FIELDS, out.tolist()))

    def l2_error(self, what: int, u=None, aux=None, t: float = 0.0) -> np.ndarray:
        """{err_h, err_hu, err_hv, combined}; aux = u_ref (DIAG_L2_REF) or VortexParams."""
        out = np.zeros(4)
        ua = None if u is None else _f64(u)
        if what == DIAG_L2_VORTEX and aux is None:
            aux = VORTEX_PARAMS
        xa = None if aux is None else _f64(aux)
        self._check(self._lib.swedg_l2_error(self._h, int(what), _p(ua), _p(xa), float(t), _p(out)))
        return out

    def diag_raw(self, what: int, u=None, aux=None, t: float = 0.0) -> bytes:
        """Raw exact accumulators of one diagnostic (merge ranks with diag_from_raw)."""
        buf = C.create_string_buffer(diag_raw_bytes())
        ua = None if u is None else _f64(u)
        if what == DIAG_L2_VORTEX and aux is None:
            aux = VORTEX_PARAMS
        xa = None if aux is None else _f64(aux)
        self._check(self._lib.swedg_diag_raw(self._h, int(what), _p(ua), _p(xa), float(t), buf))
        return buf.raw

    def sample_invariants(self, slot: int):
        self._check(self._lib.swedg_sample_invariants(self._h, int(slot)))

    def read_invariants(self, n: int) -> np.ndarray:
        out = np.zeros((n, 6))
        self._check(self._lib.swedg_read_invariants(self._h, int(n), _p(out)))
        return out

    def read_invariants_raw(self, n: int) -> bytes:
        buf = C.create_string_buffer(max(1, n * diag_raw_bytes()))
        self._check(self._lib.swedg_read_invariants_raw(self._h, int(n), buf))
        return buf.raw[: n * diag_raw_bytes()]

    def run(self, dt: float, tfinal: float, sample_every: int = 0, max_samples: int | None = None):
        """run() (run.hpp:226-262) on the resident state: returns (series [n][6], steps)."""
        nsteps = int(np.ceil(tfinal / dt - 1e-12)) if tfinal > 0 else 0
        if max_samples is None:
            cad = sample_every if sample_every > 0 else max(1, nsteps // 100)
            max_samples = nsteps // cad + 2
        series = np.zeros((max_samples, 6))
        ns = C.c_int()
        done = C.c_int()
        self._check(self._lib.swedg_run(self._h, float(dt), float(tfinal), int(sample_every), int(max_samples),
                                        _p(series), C.byref(ns), C.byref(done)))
        return series[: ns.value], done.value

    @property
    def launches(self) -> int:
        return int(self._lib.swedg_launch_count(self._h))

    @property
    def device_bytes(self) -> int:
        return int(self._lib.swedg_device_bytes(self._h))


def probe_fp64_peak(device: int = 0, reps: int = 5) -> float:
    """Measured DFMA throughput of the device, TFLOP/s (FMA = 2 flops)."""
    t = C.c_double()
    rc = lib().swedg_probe_fp64_peak(device, reps, C.byref(t))
    if rc != SWEDG_OK:
        raise SwedgError(rc, "fp64 peak probe failed")
    return t.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    rc = lib().swedg_nccl_unique_id(buf)
    if rc != SWEDG_OK:
        raise _err_class(rc)(rc, "swedg_nccl_unique_id: " + lib().swedg_create_error().decode())
    return buf.raw


def nccl_comm_init(nranks: int, uid: bytes, rank: int, device: int) -> int:
    """A library-owned NCCL communicator (ncclComm_t as int) for the halo exchange."""
    buf = C.create_string_buffer(uid, 128)
    comm = C.c_void_p()
    rc = lib().swedg_nccl_comm_init(int(nranks), buf, int(rank), int(device), C.byref(comm))
    if rc != SWEDG_OK:
        raise _err_class(rc)(rc, "swedg_nccl_comm_init: " + lib().swedg_create_error().decode())
    return comm.value


def nccl_comm_destroy(comm: int) -> None:
    lib().swedg_nccl_comm_destroy(C.c_void_p(comm))


def diag_raw_bytes() -> int:
    return int(lib().swedg_diag_raw_bytes())


def diag_from_raw(raws, n: int = 1) -> np.ndarray:
    """Merge raw records of several ranks ([rank][n] concatenated bytes) exactly and
    finish them: out [n][6]."""
    if isinstance(raws, (list, tuple)):
        raws = b"".join(raws)
    nb = diag_raw_bytes()
    nranks = len(raws) // (nb * n)
    out = np.zeros((n, 6))
    buf = C.create_string_buffer(raws, len(raws))
    rc = lib().swedg_diag_from_raw(buf, nranks, n, _p(out))
    if rc != SWEDG_OK:
        raise _err_class(rc)(rc, "swedg_diag_from_raw failed")
    return out


def ratio_kernels(Q, u, *, g: float = 9.81, nq: int | None = None, mode: int = MODE_FAST, reps: int = 5,
                  device: int = 0, outputs: bool = True):
    """bench.hpp's study kernels on the device.  Q [n][n] stored column-major ([cols][rows]),
    u [K][3][n].  Returns (t_dg_ms, t_esdg_ms, y_dg, y_esdg) (outputs None unless requested)."""
    Q = _f64(Q)
    u = _f64(u)
    K, _, n = u.shape
    y0 = np.zeros_like(u) if outputs else None
    y1 = np.zeros_like(u) if outputs else None
    t = np.zeros(2)
    rc = lib().swedg_ratio_kernels(device, n, n if nq is None else int(nq), K, _p(Q), _p(u), float(g), int(mode),
                                   int(reps), _p(y0), _p(y1), _p(t))
    if rc != SWEDG_OK:
        raise _err_class(rc)(rc, "swedg_ratio_kernels failed: " + lib().swedg_create_error().decode())
    return float(t[0]), float(t[1]), y0, y1


def exact_sum(x) -> float:
    """Host reference of the device's exact accumulator (correctly rounded sum)."""
    x = _f64(np.ravel(x))
    out = C.c_double()
    rc = lib().swedg_exact_sum(_p(x), x.size, C.byref(out))
    if rc != SWEDG_OK:
        raise _err_class(rc)(rc, "exact_sum: non-finite input")
    return out.value


def _err_class(rc: int):
    return {SWEDG_ERR_POSITIVITY: PositivityError, SWEDG_ERR_NONFINITE: NonFiniteError,
            SWEDG_ERR_INVALID: InvalidArgument}.get(rc, SwedgError)


def handle_from_case(c: dict, *, penalty: int = PENALTY_LF, mode: int = MODE_FAST,
                     device: int = 0, set_bathymetry: bool = True) -> Handle:
    """Create a handle from a case dictionary in the golden-fixture layout
    (tests/golden/*.npz: reference operators [cols][rows], per-element arrays)."""
    scheme = int(c["scheme"][0]) if np.ndim(c["scheme"]) else int(c["scheme"])
    sc = lambda k: int(np.asarray(c[k]).reshape(-1)[0])  # noqa: E731
    kw = dict(scheme=scheme, N=sc("N"), Np=sc("Np"), nq=sc("nq"), nf=sc("nf"), npf=sc("npf"),
              K=sc("K"), g=float(np.asarray(c["g"]).reshape(-1)[0]), wf=c["surfq_w"], gf=c["gf"],
              sJ=c["sJ"], nx=c["nx"], ny=c["ny"], nbr=c["nbr"], perm=c["perm"],
              penalty=penalty, mode=mode, device=device)
    if scheme == SCHEME_SBP:
        kw.update(Qr=c["sbp_Qx"], Qs=c["sbp_Qy"], face_index=c["sbp_face_index"],
                  M_diag=c["sbp_M_diag"], J_vol=c["J_vol"])
    else:
        kw.update(Qr=c["ref_Qh_x"], Qs=c["ref_Qh_y"], Vq=c["ref_Vq"], Vf=c["ref_Vf"], Pq=c["ref_Pq"],
                  Mh_inv=c["Mh_inv"])
    h = Handle(**kw)
    if set_bathymetry:
        h.set_bathymetry(c["b"])
    if "fine_w" in c and "map_coeffs" in c:
        h.set_diagnostics(w=c["fine_w"], V=c["fine_V"], Vr=c["fine_Vr"], Vs=c["fine_Vs"],
                          map_coeffs=c["map_coeffs"], Pq=c["ref_Pq"] if scheme == SCHEME_SBP else None)
    return h


# ---------------------------------------------------------------------------
# native case setup (include/swedg_setup.h)
PROBLEM_LAKE = 0
PROBLEM_VORTEX = 1
PROBLEM_DAMBREAK = 2
PROBLEM_SMOOTH = 3
PROBLEMS = {"lake": PROBLEM_LAKE, "vortex": PROBLEM_VORTEX, "dambreak": PROBLEM_DAMBREAK,
            "smooth": PROBLEM_SMOOTH}


class _CaseCfg(C.Structure):
    _fields_ = [("problem", C.c_int), ("scheme", C.c_int), ("N", C.c_int), ("nx", C.c_int),
                ("ny", C.c_int), ("warp", C.c_double), ("cfl", C.c_double), ("g", C.c_double),
                ("seed", C.c_uint), ("threads", C.c_int), ("strips", C.c_int), ("strip", C.c_int),
                ("partition", C.c_int), ("sbp_family", C.c_int), ("sbp_data_dir", C.c_char_p),
                ("sbp_rule_file", C.c_char_p)]

SBP_LEGENDRE = 0
SBP_LOBATTO = 1


PARTITION_NONE = 0
PARTITION_WEAK = 1
PARTITION_STRONG = 2


def _setup_lib():
    L = lib()
    if not getattr(L, "_setup_bound", False):
        vp = C.c_void_p
        L.swedg_case_build.argtypes = [C.POINTER(_CaseCfg), C.POINTER(vp)]
        L.swedg_case_destroy.argtypes = [vp]
        L.swedg_case_error.restype = C.c_char_p
        L.swedg_case_fill_desc.argtypes = [vp, C.POINTER(_Desc)]
        L.swedg_case_array.argtypes = [vp, C.c_char_p, C.POINTER(C.c_size_t)]
        L.swedg_case_array.restype = _dp
        L.swedg_case_iarray.argtypes = [vp, C.c_char_p, C.POINTER(C.c_size_t)]
        L.swedg_case_iarray.restype = _ip
        L.swedg_case_dt.argtypes = [vp]
        L.swedg_case_dt.restype = C.c_double
        L.swedg_case_min_edge.argtypes = [vp]
        L.swedg_case_min_edge.restype = C.c_double
        L.swedg_case_K.argtypes = [vp]
        L.swedg_sbp_rule.argtypes = [C.c_int, C.c_int, C.c_char_p, C.c_char_p, C.c_int, _ip, _ip, _dp, _dp, _dp, _ip]
        L.swedg_case_build_mesh.argtypes = [C.POINTER(_CaseCfg), _dp, C.c_int, _ip, C.c_int, _ip, C.c_int, _dp,
                                            C.c_int, C.c_int, C.POINTER(vp)]
        L._setup_bound = True
    return L


class Case:
    """A problem built by the native setup (lake / vortex / dambreak / smooth)."""

    def __init__(self, problem="smooth", *, scheme=SCHEME_HYBRIDIZED, N=4, nx=16, ny=None,
                 warp=0.0, cfl=0.125, g=0.0, seed=23, threads=0, strips=1, strip=0, scaling=None, mesh=None,
                 sbp_family=SBP_LEGENDRE, sbp_data_dir=None, sbp_rule_file=None):
        """Partitioned meshes: rank `strip`'s y-strip of P = strips, with face halos of the two
        cuts (halo_desc()).  scaling "weak": P strips of ny rows of a global nx x (ny P) mesh on
        the problem's domain stretched P times in y (fixed work per rank; the default when
        strips > 1); "strong": the problem's nx x ny mesh cut into P strips of ny/P rows
        (strips = 1 with scaling "strong": one rank whose halos are its own periodic cut).
        strip = -1: the whole global mesh in one piece.
        mesh: a caller-supplied mesh instead (dict with verts [nv][2], tris [ne][3],
        wall_faces [nw][2], domain (xc, yc, Lx, Ly), periodic_x, periodic_y; e.g. from
        io.read_mesh_text) — swedg_case_build_mesh."""
        L = _setup_lib()
        cfg = _CaseCfg()
        cfg.problem = PROBLEMS[problem] if isinstance(problem, str) else int(problem)
        cfg.scheme, cfg.N, cfg.nx, cfg.ny = scheme, N, nx, ny if ny is not None else nx
        cfg.warp, cfg.cfl, cfg.g, cfg.seed, cfg.threads = warp, cfl, g, seed, threads
        cfg.strips, cfg.strip = strips, strip
        cfg.partition = {None: PARTITION_NONE, "weak": PARTITION_WEAK, "strong": PARTITION_STRONG}[scaling]
        cfg.sbp_family = sbp_family
        cfg.sbp_data_dir = sbp_data_dir.encode() if sbp_data_dir else None
        cfg.sbp_rule_file = sbp_rule_file.encode() if sbp_rule_file else None
        h = C.c_void_p()
        if mesh is None:
            rc = L.swedg_case_build(C.byref(cfg), C.byref(h))
        else:
            v = _f64(mesh["verts"]).reshape(-1, 2)
            t = _i32(mesh["tris"]).reshape(-1, 3)
            w = _i32(mesh.get("wall_faces", np.zeros((0, 2)))).reshape(-1, 2)
            dom = _f64(mesh["domain"])
            rc = L.swedg_case_build_mesh(C.byref(cfg), _p(v), len(v), _pi(t), len(t), _pi(w) if len(w) else None,
                                         len(w), _p(dom), int(mesh.get("periodic_x", 0)),
                                         int(mesh.get("periodic_y", 0)), C.byref(h))
        if rc != SWEDG_OK:
            raise _err_class(rc)(rc, "swedg_case_build: " + L.swedg_case_error().decode())
        self._c, self._lib = h, L
        self.scheme, self.N = scheme, N
        self.problem = problem if isinstance(problem, str) else None
        self.desc = _Desc()
        L.swedg_case_fill_desc(self._c, C.byref(self.desc))
        d = self.desc
        self.K, self.Np, self.nq, self.nf, self.npf = d.K, d.Np, d.nq, d.nf, d.npf
        self.g = d.g
        self.dt = L.swedg_case_dt(self._c)
        self.min_edge = L.swedg_case_min_edge(self._c)
        self.nstate = self.nq if scheme == SCHEME_SBP else self.Np
        self.n_halo = d.n_halo
        self.nx = nx

    def array(self, name: str) -> np.ndarray:
        n = C.c_size_t()
        p = self._lib.swedg_case_array(self._c, name.encode(), C.byref(n))
        if not p:
            raise KeyError(name)
        return np.ctypeslib.as_array(p, shape=(n.value,)).copy() if n.value else np.zeros(0)

    def iarray(self, name: str) -> np.ndarray:
        n = C.c_size_t()
        p = self._lib.swedg_case_iarray(self._c, name.encode(), C.byref(n))
        if not p:
            raise KeyError(name)
        return np.ctypeslib.as_array(p, shape=(n.value,)).copy() if n.value else np.zeros(0, np.int32)

    def view(self, name: str, integer: bool = False) -> np.ndarray:
        """Zero-copy view of a named case array (valid while the case is alive)."""
        n = C.c_size_t()
        f = self._lib.swedg_case_iarray if integer else self._lib.swedg_case_array
        p = f(self._c, name.encode(), C.byref(n))
        if not p:
            raise KeyError(name)
        return np.ctypeslib.as_array(p, shape=(n.value,))

    def u0(self) -> np.ndarray:
        return self.array("u0").reshape(self.K, 3, self.nstate)

    def b(self) -> np.ndarray:
        return self.array("b").reshape(self.K, self.nstate)

    def halo_desc(self) -> dict | None:
        """The halo exchange map of a partitioned case (swedg_case_fill_halo), else None."""
        if self.n_halo == 0:
            return None
        return {k: self.iarray("halo_" + k) for k in ("send_peer", "send_count", "send_elem", "send_face",
                                                     "recv_peer", "recv_count")}

    def handle(self, *, penalty=PENALTY_LF, mode=MODE_FAST, device=0, set_bathymetry=True,
               diagnostics=True) -> "Handle":
        h = Handle.from_desc(self.desc, self, penalty=penalty, mode=mode, device=device,
                             b=self.b() if set_bathymetry else None)
        if diagnostics:
            h.set_diagnostics(**self.diag_arrays())
        halo = self.halo_desc()
        if halo is not None:
            h.set_halo(halo)
        return h

    def diag_arrays(self) -> dict:
        """FineQuad(N) operators and mapping coefficients (diagnostics.hpp:142-165)."""
        d = dict(w=self.array("fine_w"), V=self.array("fine_V"), Vr=self.array("fine_Vr"),
                 Vs=self.array("fine_Vs"), map_coeffs=self.array("map_coeffs"))
        if self.scheme == SCHEME_SBP:
            d["Pq"] = self.array("Pq")
        return d

    def close(self):
        if getattr(self, "_c", None):
            self._lib.swedg_case_destroy(self._c)
            self._c = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def sbp_rule(N: int, family: int = SBP_LEGENDRE, data_dir: str | None = None, rule_file: str | None = None):
    """sbp_rule / load_sbp_rule_file (quadrature.hpp:290-343) through the native setup:
    dict(x, y, w, npf, face_index).  Raises InvalidArgument with the reference's message."""
    L = _setup_lib()
    mx = 512
    x, y, w = np.zeros(mx), np.zeros(mx), np.zeros(mx)
    fi = np.zeros(mx, dtype=np.int32)
    nq, npf = C.c_int(), C.c_int()
    rc = L.swedg_sbp_rule(int(N), int(family), data_dir.encode() if data_dir else None,
                          rule_file.encode() if rule_file else None, mx, C.byref(nq), C.byref(npf), _p(x), _p(y),
                          _p(w), _pi(fi))
    if rc != SWEDG_OK:
        raise _err_class(rc)(rc, L.swedg_case_error().decode())
    n = nq.value
    return {"x": x[:n].copy(), "y": y[:n].copy(), "w": w[:n].copy(), "npf": npf.value,
            "face_index": fi[:3 * npf.value].copy()}


def _handle_from_desc(cls, desc, owner, *, penalty=PENALTY_LF, mode=MODE_FAST, device=0, b=None):
    L = lib()
    d = _Desc()
    C.pointer(d)[0] = desc
    d.penalty, d.mode, d.device = penalty, mode, device
    h = C.c_void_p()
    rc = L.swedg_create(C.byref(d), C.byref(h))
    if rc != SWEDG_OK:
        raise _err_class(rc)(rc, "swedg_create: " + L.swedg_create_error().decode())
    self = cls.__new__(cls)
    self._h, self._lib = h, L
    self.sizes = Sizes(d.N, d.Np, d.nq, d.nf, d.npf, d.K)
    self.scheme = d.scheme
    self.nstate = d.nq if d.scheme == SCHEME_SBP else d.Np
    self._owner = owner
    if b is not None:
        self.set_bathymetry(b)
    return self


Handle.from_desc = classmethod(_handle_from_desc)
