"""ctypes binding of the C oracle (oracle/swedg_oracle.c -> oracle/liboracle.so).

TEST INFRASTRUCTURE: the checker the CUDA path is compared against.  Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(REPO, "oracle", "liboracle.so")
LIB_LD = os.path.join(REPO, "oracle", "liboracle_ld.so")  # same code, long double arithmetic
GOLDEN = os.path.join(REPO, "tests", "golden")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class OracleOps(C.Structure):
    _fields_ = [
        ("N", C.c_int), ("Np", C.c_int), ("nq", C.c_int), ("nf", C.c_int), ("npf", C.c_int),
        ("K", C.c_int), ("scheme", C.c_int), ("penalty_lf", C.c_int), ("g", C.c_double),
        ("Vq", _dp), ("Vf", _dp), ("Pq", _dp), ("Qr", _dp), ("Qs", _dp), ("wf", _dp),
        ("face_index", _ip), ("gf", _dp), ("sJ", _dp), ("nx", _dp), ("ny", _dp),
        ("Mh_inv", _dp), ("J_vol", _dp), ("M_diag", _dp), ("nbr", _ip), ("perm", _ip),
        ("b_stacked", _dp), ("src_x", _dp), ("src_y", _dp),
    ]


def _build_lib(path, extra) -> None:
    src = os.path.join(REPO, "oracle", "swedg_oracle.c")
    if not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        subprocess.run(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                        "-shared"] + extra + [src, "-o", path, "-lm"], check=True)


_libs = {}


def lib(precision: str = "double"):
    if precision not in _libs:
        path, extra = (LIB, []) if precision == "double" else (LIB_LD, ["-DORACLE_LONG_DOUBLE"])
        _build_lib(path, extra)
        _lib = C.CDLL(path)
        _lib.oracle_set_bathymetry.argtypes = [C.POINTER(OracleOps), _dp, _dp, _dp, _dp]
        _lib.oracle_entropy_projection.argtypes = [C.POINTER(OracleOps), _dp, _dp, _ip]
        _lib.oracle_rhs_from_proj.argtypes = [C.POINTER(OracleOps), _dp, _dp, _ip, C.c_int, _ip]
        _lib.oracle_rhs.argtypes = [C.POINTER(OracleOps), _dp, _dp, _dp, _ip]
        _lib.oracle_rhs_sbp.argtypes = [C.POINTER(OracleOps), _dp, _dp, _ip, C.c_int, _ip]
        _lib.oracle_step_lsrk45.argtypes = [C.POINTER(OracleOps), _dp, _dp, C.c_double, C.c_int, _ip]
        _lib.oracle_rhs_subset.argtypes = [C.POINTER(OracleOps), _dp, _dp, _ip, C.c_int, _ip]
        _lib.oracle_rhs_from_proj_n.argtypes = [C.POINTER(OracleOps), _dp, C.c_int, _dp, _ip, C.c_int, _ip]
        _lib.oracle_ratio_matvec.argtypes = [C.c_int, C.c_int, _dp, _dp, C.c_double, _dp]
        _lib.oracle_ratio_fluxdiff.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_double, _dp]
        _lib.oracle_project_nodal.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp]
        _lib.oracle_diag.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                     C.c_double, C.c_double, C.c_int, _dp, _dp, _dp, C.POINTER(C.c_long)]
        _libs[precision] = _lib
    return _libs[precision]


def _p(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _pi(a):
    return None if a is None else a.ctypes.data_as(_ip)


def load_golden(name: str) -> dict:
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return {k: z[k] for k in z.files}


class Oracle:
    """The C restatement driven from a case dictionary (golden fixture layout)."""

    def __init__(self, case: dict, penalty_lf: bool = True, precision: str = "double"):
        """precision "double" = the reference's arithmetic (bitwise); "ld" = the same
        algorithm in x87 long double (an accuracy yardstick, not a parity target)."""
        self.L = lib(precision)
        c = {k: np.ascontiguousarray(v) for k, v in case.items()}
        self.c = c
        self.scheme = int(c["scheme"][0])
        sc = self.scheme
        op = OracleOps()
        op.N = int(c["N"][0])
        op.Np = int(c["Np"][0])
        op.nq = int(c["nq"][0])
        op.nf = int(c["nf"][0])
        op.npf = int(c["npf"][0])
        op.K = int(c["K"][0])
        op.scheme = sc
        op.penalty_lf = 1 if penalty_lf else 0
        op.g = float(c["g"][0])
        # reference operators stored [cols][rows] == column-major
        self._keep = []

        def keep(a, dt=np.float64):
            a = np.ascontiguousarray(a, dtype=dt)
            self._keep.append(a)
            return a

        op.Vq = _p(keep(c["ref_Vq"]))
        op.Vf = _p(keep(c["ref_Vf"]))
        op.Pq = _p(keep(c["ref_Pq"]))
        if sc == 1:
            op.Qr = _p(keep(c["sbp_Qx"]))
            op.Qs = _p(keep(c["sbp_Qy"]))
            op.face_index = _pi(keep(c["sbp_face_index"], np.int32))
            op.M_diag = _p(keep(c["sbp_M_diag"]))
            op.J_vol = _p(keep(c["J_vol"]))
        else:
            op.Qr = _p(keep(c["ref_Qh_x"]))
            op.Qs = _p(keep(c["ref_Qh_y"]))
            op.Mh_inv = _p(keep(c["Mh_inv"]))
        op.wf = _p(keep(c["surfq_w"]))
        op.gf = _p(keep(c["gf"]))
        op.sJ = _p(keep(c["sJ"]))
        op.nx = _p(keep(c["nx"]))
        op.ny = _p(keep(c["ny"]))
        op.nbr = _pi(keep(c["nbr"], np.int32))
        op.perm = _pi(keep(c["perm"], np.int32))
        self.op = op
        self.K, self.nq, self.nf, self.Np = op.K, op.nq, op.nf, op.Np
        self.nh = op.nq + op.nf
        self.set_bathymetry(c["b"])

    def set_bathymetry(self, b):
        b = np.ascontiguousarray(b, dtype=np.float64)
        K = self.K
        if self.scheme == 1:
            self.b_stacked = np.zeros((K, self.nq))
            self.src_x = np.zeros((K, self.nq))
            self.src_y = np.zeros((K, self.nq))
        else:
            self.b_stacked = np.zeros((K, self.nh))
            self.src_x = np.zeros((K, self.nh))
            self.src_y = np.zeros((K, self.nh))
        self.L.oracle_set_bathymetry(C.byref(self.op), _p(b), _p(self.b_stacked), _p(self.src_x),
                                    _p(self.src_y))
        self.op.b_stacked = _p(self.b_stacked)
        self.op.src_x = _p(self.src_x)
        self.op.src_y = _p(self.src_y)

    def entropy_projection(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        proj = np.zeros((self.K, 3, self.nh))
        bad = C.c_int(-1)
        err = self.L.oracle_entropy_projection(C.byref(self.op), _p(u), _p(proj), C.byref(bad))
        return proj, err, bad.value

    def rhs(self, u, elems=None):
        u = np.ascontiguousarray(u, dtype=np.float64)
        bad = C.c_int(-1)
        if self.scheme == 1:
            du = np.zeros((self.K, 3, self.nq))
            ei = None if elems is None else np.ascontiguousarray(elems, dtype=np.int32)
            err = self.L.oracle_rhs_sbp(C.byref(self.op), _p(u), _p(du), _pi(ei),
                                       0 if ei is None else len(ei), C.byref(bad))
            return du, err, bad.value
        du = np.zeros((self.K, 3, self.Np))
        ei = None if elems is None else np.ascontiguousarray(elems, dtype=np.int32)
        err = self.L.oracle_rhs_subset(C.byref(self.op), _p(u), _p(du), _pi(ei),
                                       0 if ei is None else len(ei), C.byref(bad))
        return du, err, bad.value

    def rhs_from_proj(self, proj_all):
        """du of the K owned elements from projections of owned + halo element slots
        (proj_all: [K + n_halo][3][nh]; nbr may address the halo slots)."""
        proj_all = np.ascontiguousarray(proj_all, dtype=np.float64)
        du = np.zeros((self.K, 3, self.Np))
        bad = C.c_int(-1)
        ei = np.arange(self.K, dtype=np.int32)
        err = self.L.oracle_rhs_from_proj_n(C.byref(self.op), _p(proj_all), int(proj_all.shape[0]), _p(du),
                                            _pi(ei), self.K, C.byref(bad))
        return du, err, bad.value

    def step_lsrk45(self, u, res, dt, nsteps):
        u = np.array(u, dtype=np.float64, copy=True)
        res = np.array(res, dtype=np.float64, copy=True)
        bad = C.c_int(-1)
        err = self.L.oracle_step_lsrk45(C.byref(self.op), _p(u), _p(res), float(dt), int(nsteps),
                                       C.byref(bad))
        return u, res, err


VORTEX_PARAMS = np.array([1.0, 1.0, 0.0, 5.0, 2.0, 0.0, 0.0])  # VortexParams defaults (diagnostics.hpp:30-38)


def project_nodal(Pq, u_nodal):
    """Pq * u per element, k-ascending (diagnostics.hpp:226-230); u_nodal [K][ncol][nq]."""
    u_nodal = np.ascontiguousarray(u_nodal, dtype=np.float64)
    Pq = np.ascontiguousarray(Pq, dtype=np.float64)  # [nq][Np] == Np x nq column-major
    K, ncol, nq = u_nodal.shape
    Np = Pq.shape[1]
    out = np.zeros((K, ncol, Np))
    lib().oracle_project_nodal(K, Np, nq, ncol, _p(Pq), _p(u_nodal), _p(out))
    return out


def diag(fine, u_modal, *, what, b_modal=None, u_ref=None, t=0.0, g=0.0, vortex=VORTEX_PARAMS):
    """Per-point terms [K][nfine][4] and the reference's serial sums of compute_invariants
    (what=0), l2_error vs a discrete state (1) or vs the vortex (2).  fine: dict with
    fine_w, fine_V, fine_Vr, fine_Vs ([Np][nfine] = column-major) and map_coeffs [K][2][Np].
    Returns (terms, sums, min_h, err, bad_elem)."""
    f = {k: np.ascontiguousarray(fine[k], dtype=np.float64) for k in
         ("fine_w", "fine_V", "fine_Vr", "fine_Vs", "map_coeffs")}
    u = np.ascontiguousarray(u_modal, dtype=np.float64)
    K, _, Np = u.shape
    nf = f["fine_w"].shape[0]
    b = None if b_modal is None else np.ascontiguousarray(b_modal, dtype=np.float64)
    ur = None if u_ref is None else np.ascontiguousarray(u_ref, dtype=np.float64)
    vp = np.ascontiguousarray(vortex, dtype=np.float64)
    terms = np.zeros((K, nf, 4))
    sums = np.zeros(4)
    mh = C.c_double(0.0)
    bad = C.c_long(-1)
    err = lib().oracle_diag(K, Np, nf, _p(f["fine_w"]), _p(f["fine_V"]), _p(f["fine_Vr"]), _p(f["fine_Vs"]),
                            _p(f["map_coeffs"]), _p(u), _p(b), _p(ur), _p(vp), float(t), float(g), int(what),
                            _p(terms), _p(sums), C.byref(mh), C.byref(bad))
    return terms, sums, mh.value, err, bad.value


def ratio_kernels(Q, u, g=9.81, nq=None):
    """bench.hpp kernel_matvec and kernel_fluxdiff(_skew): Q [n][n] as stored ([cols][rows]),
    u [K][3][n].  Returns (y_dg, y_esdg)."""
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    K, _, n = u.shape
    y_dg = np.zeros((K, 3, n))
    y_es = np.zeros((K, 3, n))
    L = lib()
    L.oracle_ratio_matvec(n, K, _p(Q), _p(u), float(g), _p(y_dg))
    L.oracle_ratio_fluxdiff(n, n if nq is None else int(nq), K, _p(Q), _p(u), float(g), _p(y_es))
    return y_dg, y_es


def case_dict(c) -> dict:
    """A native-setup case (paper_2005_02516_b200.capi.Case) in the golden-fixture layout."""
    d = {"scheme": [c.scheme], "N": [c.N], "Np": [c.Np], "nq": [c.nq], "nf": [c.nf], "npf": [c.npf],
         "K": [c.K], "g": [c.g], "surfq_w": c.array("surfq_w"), "gf": c.array("gf"), "sJ": c.array("sJ"),
         "nx": c.array("nx"), "ny": c.array("ny"), "nbr": c.iarray("nbr"), "perm": c.iarray("perm"),
         "b": c.b(), "u": c.u0(), "ref_Vq": c.array("Vq"), "ref_Vf": c.array("Vf"), "ref_Pq": c.array("Pq")}
    if c.scheme == 1:
        d.update(sbp_Qx=c.array("Qr"), sbp_Qy=c.array("Qs"), sbp_face_index=c.iarray("face_index"),
                 sbp_M_diag=c.array("M_diag"), J_vol=c.array("J_vol"))
    else:
        d.update(ref_Qh_x=c.array("Qr"), ref_Qh_y=c.array("Qs"), Mh_inv=c.array("Mh_inv"))
    return {k: np.asarray(v) for k, v in d.items()}
