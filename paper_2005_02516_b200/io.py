"""Input/output formats around the solver, byte-compatible
with the reference's writers:

  mesh text     read_mesh_text / write_mesh_text         mesh.hpp:462-493
  CSV           write_invariants_csv / write_errors_csv  diagnostics.hpp:289-316
  legacy VTK    write_solution_vtk                       diagnostics.hpp:318-375

Host-side formatting only; the numbers come from the device (capi.Handle
diagnostics / get_state) or from the native setup (capi.Case arrays).  Files are
written atomically (temporary file + rename, diagnostics.hpp:272-285).
"""
from __future__ import annotations

import math
import os

import numpy as np


# ---- mesh text (mesh.hpp:462-493) --------------------------------------------
def write_mesh_text(verts, tris, wall_faces=()) -> str:
    """Header "nv ne", vertex lines "x y" (17 significant digits), element lines
    "v0 v1 v2", then "wallface e f" records."""
    verts = np.asarray(verts, dtype=np.float64).reshape(-1, 2)
    tris = np.asarray(tris, dtype=np.int64).reshape(-1, 3)
    out = [f"{len(verts)} {len(tris)}\n"]
    out += [f"{x:.17g} {y:.17g}\n" for x, y in verts.tolist()]
    out += [f"{a} {b} {c}\n" for a, b, c in tris.tolist()]
    out += [f"wallface {e} {f}\n" for e, f in np.asarray(wall_faces, dtype=np.int64).reshape(-1, 2).tolist()]
    return "".join(out)


def read_mesh_text(text: str) -> dict:
    """Parse the text format; errors mirror the reference's runtime_error messages."""
    tok = text.split()
    pos = 0

    def take(n, what):
        nonlocal pos
        if pos + n > len(tok):
            raise ValueError(what)
        v = tok[pos:pos + n]
        pos += n
        return v

    try:
        nv, ne = (int(x) for x in take(2, "bad mesh header"))
    except ValueError:
        raise ValueError("bad mesh header") from None
    verts = np.empty((nv, 2))
    for i in range(nv):
        try:
            verts[i] = [float(x) for x in take(2, "bad vertex line")]
        except ValueError:
            raise ValueError("bad vertex line") from None
    tris = np.empty((ne, 3), dtype=np.int32)
    for e in range(ne):
        try:
            tris[e] = [int(x) for x in take(3, "bad element line")]
        except ValueError:
            raise ValueError("bad element line") from None
    walls = []
    while pos < len(tok):
        t = tok[pos]
        pos += 1
        if t != "wallface":
            raise ValueError("unknown mesh record " + t)
        walls.append([int(x) for x in take(2, "bad wallface record")])
    return {"verts": verts, "tris": tris, "wall_faces": np.asarray(walls, dtype=np.int32).reshape(-1, 2)}


# ---- CSV (diagnostics.hpp:286-316) -----------------------------------------------
def csv_number(v: float) -> str:
    return "%.17g" % v


def write_file_atomic(path: str, content: str) -> None:
    d = os.path.dirname(path)
    if d:
        os.makedirs(d, exist_ok=True)
    tmp = path + ".tmp"
    with open(tmp, "w", newline="") as f:
        f.write(content)
    os.replace(tmp, path)


def invariants_csv(series) -> str:
    """series: rows (t, mass, momentum_x, momentum_y, entropy, min_h)."""
    out = ["t,mass,momentum_x,momentum_y,entropy,min_h\n"]
    for row in np.asarray(series, dtype=np.float64).reshape(-1, 6).tolist():
        out.append(",".join(csv_number(v) for v in row) + "\n")
    return "".join(out)


def write_invariants_csv(path: str, series) -> None:
    write_file_atomic(path, invariants_csv(series))


def errors_csv(reports, orders=()) -> str:
    """reports: rows (N, h_mesh, err_h, err_hu, err_hv, combined); orders[i] (may be
    shorter or non-finite: empty field)."""
    out = ["N,h_mesh,err_h,err_hu,err_hv,err_combined,order\n"]
    for i, r in enumerate(np.asarray(reports, dtype=np.float64).reshape(-1, 6).tolist()):
        line = f"{int(r[0])}," + ",".join(csv_number(v) for v in r[1:]) + ","
        if i < len(orders) and math.isfinite(orders[i]):
            line += csv_number(orders[i])
        out.append(line + "\n")
    return "".join(out)


def write_errors_csv(path: str, reports, orders=()) -> None:
    write_file_atomic(path, errors_csv(reports, orders))


# ---- legacy VTK (diagnostics.hpp:318-375) -------------------------------------------
def _lattice_subtriangles(N: int):
    def idx(i, j):
        return i * (N + 1) - i * (i - 1) // 2 + j

    sub = []
    for i in range(N):
        for j in range(N - i):
            sub.append((idx(i, j), idx(i + 1, j), idx(i, j + 1)))
            if j < N - i - 1:
                sub.append((idx(i + 1, j), idx(i + 1, j + 1), idx(i, j + 1)))
    return sub


def _lattice_values(Vl, coeffs):
    """Vl * c per element with the reference's k-ascending sums (no contraction):
    Vl [Np][Np] stored column-major ([cols][rows]); coeffs [K][Np] -> [K][Np]."""
    Vl = np.asarray(Vl, dtype=np.float64)
    K, Np = coeffs.shape
    acc = np.zeros((K, Np))
    for m in range(Np):
        acc = acc + Vl[m][None, :] * coeffs[:, m][:, None]
    return acc


def solution_vtk(map_nodes, N: int, u_modal, b_modal, lattice_V) -> str:
    """map_nodes [K][2][Np], u_modal [K][3][Np], b_modal [K][Np], lattice_V = basis at the
    mapping lattice (capi.Case.array("lattice_V"), column-major Np x Np)."""
    Np = (N + 1) * (N + 2) // 2
    mn = np.asarray(map_nodes, dtype=np.float64).reshape(-1, 2, Np)
    u = np.asarray(u_modal, dtype=np.float64).reshape(-1, 3, Np)
    b = np.asarray(b_modal, dtype=np.float64).reshape(-1, Np)
    Vl = np.asarray(lattice_V, dtype=np.float64).reshape(Np, Np)
    K = mn.shape[0]
    sub = _lattice_subtriangles(N)
    out = ["# vtk DataFile Version 3.0\nshallow water solution\nASCII\nDATASET UNSTRUCTURED_GRID\n",
           f"POINTS {K * Np} double\n"]
    for k in range(K):
        for x, y in zip(mn[k, 0].tolist(), mn[k, 1].tolist()):
            out.append(f"{x:.15g} {y:.15g} 0\n")
    nc = K * len(sub)
    out.append(f"CELLS {nc} {4 * nc}\n")
    for k in range(K):
        for s in sub:
            out.append(f"3 {k * Np + s[0]} {k * Np + s[1]} {k * Np + s[2]}\n")
    out.append(f"CELL_TYPES {nc}\n")
    out.append("5\n" * nc)
    out.append(f"POINT_DATA {K * Np}\n")
    hv = _lattice_values(Vl, u[:, 0])
    huv = _lattice_values(Vl, u[:, 1])
    hvv = _lattice_values(Vl, u[:, 2])
    bv = _lattice_values(Vl, b)
    for name, arr in (("H", hv + bv), ("h", hv), ("hu", huv), ("hv", hvv), ("b", bv)):
        out.append(f"SCALARS {name} double 1\nLOOKUP_TABLE default\n")
        out.append("".join(f"{v:.15g}\n" for v in arr.ravel().tolist()))
    return "".join(out)


def write_solution_vtk(path: str, map_nodes, N: int, u_modal, b_modal, lattice_V) -> None:
    write_file_atomic(path, solution_vtk(map_nodes, N, u_modal, b_modal, lattice_V))
