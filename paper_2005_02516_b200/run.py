"""run() (run.hpp:226-284) on the device: the reference's time loop with invariant
sampling, the final L2 error and the optional output files, over the C ABI.

    from paper_2005_02516_b200 import capi, run
    case = capi.Case("vortex", N=3, nx=16)
    res = run.run(case, tfinal=0.5, out_dir="out")   # invariants.csv, errors.csv, solution_*.vtk

The state stays on the device for the whole integration (swedg_run: graph-
replayed steps, device-side invariant samples); the host sees it only for the
output files and the result.
"""
from __future__ import annotations

import os

import numpy as np

from . import capi
from . import io as sio


def _project(Pq, u):
    """Pq * u per element, k-ascending sums (project_nodal, diagnostics.hpp:226-230).
    Pq stored column-major [nq][Np]; u [K][c][nq] -> [K][c][Np]."""
    Pq = np.asarray(Pq, dtype=np.float64)
    nq, Np = Pq.shape
    K, ncol, _ = u.shape
    acc = np.zeros((K, ncol, Np))
    for q in range(nq):
        acc = acc + Pq[q][None, None, :] * u[:, :, q][:, :, None]
    return acc


def modal_solution(case, u):
    """Case::modal_solution (run.hpp:65-68): the state itself, or Pq * nodal state for SBP."""
    if case.scheme != capi.SCHEME_SBP:
        return np.asarray(u)
    return _project(case.array("Pq").reshape(case.nq, case.Np), np.asarray(u))


def modal_bathymetry(case):
    """Case::modal_bathymetry (run.hpp:69-74)."""
    b = case.b()
    if case.scheme != capi.SCHEME_SBP:
        return b
    return _project(case.array("Pq").reshape(case.nq, case.Np), b[:, None, :])[:, 0, :]


def run(case, *, tfinal: float, handle=None, mode: int = capi.MODE_FAST, sample_every: int = 0,
        out_dir: str | None = None, problem: str | None = None) -> dict:
    """Integrate the case's initial state to tfinal (run.hpp:226-284).  problem selects
    the error norm like the reference's builders: "lake" (vs the discrete initial
    state), "vortex" (vs vortex_exact), otherwise none; default: the case's problem."""
    problem = problem or getattr(case, "problem", None)
    h = handle or case.handle(mode=mode)
    u0 = case.u0()
    h.set_state(u0, None, 0.0)
    N = case.N
    Vl = case.array("lattice_V") if out_dir else None
    mn = case.array("map_nodes") if out_dir else None
    bm = modal_bathymetry(case)
    if out_dir:
        sio.write_solution_vtk(os.path.join(out_dir, "solution_0.vtk"), mn, N, modal_solution(case, u0), bm, Vl)
    series, steps = h.run(case.dt, tfinal, sample_every)
    u, _, t = h.get_state(with_res=False)
    err = None
    if problem == "lake":
        e = h.l2_error(capi.DIAG_L2_REF, None, modal_solution(case, u0), t)
    elif problem == "vortex":
        vp = list(capi.VORTEX_PARAMS)
        vp[4] = case.g
        e = h.l2_error(capi.DIAG_L2_VORTEX, None, vp, t)
    else:
        e = None
    if e is not None:
        err = {"N": N, "h_mesh": case.min_edge, "err_h": e[0], "err_hu": e[1], "err_hv": e[2], "combined": e[3]}
    if out_dir:
        sio.write_invariants_csv(os.path.join(out_dir, "invariants.csv"), series)
        if err:
            sio.write_errors_csv(os.path.join(out_dir, "errors.csv"),
                                 [[N, err["h_mesh"], err["err_h"], err["err_hu"], err["err_hv"], err["combined"]]])
        sio.write_solution_vtk(os.path.join(out_dir, "solution_%g.vtk" % t), mn, N, modal_solution(case, u), bm, Vl)
    if handle is None:
        h.close()
    return {"series": series, "steps": steps, "dt": case.dt, "t": t, "error": err, "u": u}


def convergence_study(problem: str, degrees, levels: int, *, nx: int = 8, ny: int = 4, warp: float = 0.0,
                      scheme: int = capi.SCHEME_HYBRIDIZED, tfinal: float = 0.5, mode: int = capi.MODE_FAST,
                      cfl: float = 0.125) -> list:
    """convergence_study (run.hpp:287-332): for each degree, `levels` meshes doubling nx
    and ny, run() to tfinal and the observed order log2(e_prev / e) of the combined
    L2 error.  Rows: dict(N, nx, ny, error, order)."""
    import math

    rows = []
    for N in degrees:
        prev = None
        for lev in range(levels):
            c = capi.Case(problem, scheme=scheme, N=N, nx=nx << lev, ny=ny << lev, warp=warp, cfl=cfl)
            res = run(c, tfinal=tfinal, mode=mode, problem=problem)
            err = res["error"]
            order = math.log2(prev["combined"] / err["combined"]) if prev else float("nan")
            rows.append({"N": N, "nx": nx << lev, "ny": ny << lev, "error": err, "order": order})
            prev = err
            c.close()
    return rows
