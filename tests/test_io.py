"""Output formats and mesh import (mesh.hpp:462-493,
diagnostics.hpp:272-375): byte-for-byte against the reference's own writers
(tests/golden/io.npz, written by the unmodified reference), and a case built from
an imported mesh text equal, array for array, to the reference's case on the same
mesh.  CPU only."""
import numpy as np
import pytest

from oracle_py import load_golden
from paper_2005_02516_b200 import capi
from paper_2005_02516_b200 import io as sio


def text(a):
    return bytes(np.asarray(a).astype(np.uint8)).decode()


G = load_golden("io")


@pytest.mark.parametrize("key", ["mesh_lake_text", "mesh_dam_text"])
def test_mesh_text_round_trip_bytes(key):
    src = text(G[key])
    m = sio.read_mesh_text(src)
    assert sio.write_mesh_text(m["verts"], m["tris"], m["wall_faces"]) == src
    if key == "mesh_dam_text":
        assert len(m["wall_faces"]) > 0


def test_mesh_text_errors():
    with pytest.raises(ValueError, match="bad mesh header"):
        sio.read_mesh_text("x 3")
    with pytest.raises(ValueError, match="bad vertex line"):
        sio.read_mesh_text("3 1\n0 0\n1 0\n")
    with pytest.raises(ValueError, match="bad element line"):
        sio.read_mesh_text("3 1\n0 0\n1 0\n0 1\n0 1\n")
    with pytest.raises(ValueError, match="unknown mesh record"):
        sio.read_mesh_text("3 1\n0 0\n1 0\n0 1\n0 1 2\nwall 0 1\n")


def test_csv_writers_bytes(tmp_path):
    sio.write_invariants_csv(str(tmp_path / "invariants.csv"), G["series"])
    assert (tmp_path / "invariants.csv").read_text() == text(G["invariants_csv"])
    sio.write_errors_csv(str(tmp_path / "e" / "errors.csv"), [G["error"]], [])
    assert (tmp_path / "e" / "errors.csv").read_text() == text(G["errors_csv"])
    assert not list(tmp_path.glob("*.tmp"))


def test_vtk_writer_bytes():
    c = capi.Case("vortex", N=2, nx=4)
    Vl = c.array("lattice_V")
    assert sio.solution_vtk(G["vtk_map_nodes"], 2, G["u0"], G["b"], Vl) == text(G["vtk0_text"])
    assert sio.solution_vtk(G["vtk_map_nodes"], 2, G["u_final"], G["b"], Vl) == text(G["vtk1_text"])
    # the native setup's own mapping nodes give the same file
    assert sio.solution_vtk(c.array("map_nodes"), 2, c.u0(), c.b(), Vl) == text(G["vtk0_text"])


def test_case_from_imported_mesh_equals_reference_case():
    """The reference's unwarped 8 x 8 lake mesh as text -> swedg_case_build_mesh with the lake
    problem, N=3, warp 0.1, periodic: every setup array bit-for-bit the reference's C2 case
    (tests/golden/c2_lake.npz: uniform mesh, set_mapping_degree, warp_mesh, build_lake_case)."""
    m = sio.read_mesh_text(text(G["mesh_lake_text"]))
    mesh = dict(m, domain=(0.0, 0.0, 2.0, 2.0), periodic_x=1, periodic_y=1)
    c = capi.Case("lake", N=3, warp=0.1, mesh=mesh)
    ref = load_golden("c2_lake")
    assert c.K == int(ref["K"][0])
    K = c.K
    for name, key in (("gf", "gf"), ("sJ", "sJ"), ("nx", "nx"), ("J_vol", "J_vol"), ("Mh_inv", "Mh_inv"),
                      ("map_nodes", "map_nodes")):
        np.testing.assert_array_equal(c.array(name).reshape(K, -1), ref[key].reshape(K, -1), err_msg=name)
    np.testing.assert_array_equal(c.u0(), ref["u"])
    np.testing.assert_array_equal(c.b(), ref["b"])
    np.testing.assert_array_equal(c.iarray("perm").reshape(K, -1), ref["perm"].reshape(K, -1))
    assert c.dt == float(ref["dt"][0])


def test_imported_mesh_walls_and_open_boundaries():
    """Dam-break mesh text (wall faces on the dam) without periodicity: every open boundary
    face and every tagged face becomes a wall."""
    m = sio.read_mesh_text(text(G["mesh_dam_text"]))
    mesh = dict(m, domain=(0.0, 0.0, 20.0, 20.0), periodic_x=0, periodic_y=0)
    c = capi.Case("dambreak", N=2, cfl=0.0625, mesh=mesh)
    nbr = c.iarray("nbr").reshape(c.K, 3)
    for e, f in m["wall_faces"]:
        assert nbr[e, f] == -1
    assert (nbr == -1).sum() >= 4 * 6 + len(m["wall_faces"])
