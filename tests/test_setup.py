"""The native case setup (csrc/setup.cpp via include/swedg_setup.h) against the
reference's own setup outputs (tests/golden/*.npz), CPU only.

The setup restates quadrature / refelem / mesh / geometry / connectivity /
precompute_element_ops / make_state with the oracle build's evaluation order,
so every array is asserted BIT-FOR-BIT equal to the reference's."""
import numpy as np
import pytest

from oracle_py import load_golden
from paper_2005_02516_b200 import capi

CASES = [
    # golden name, problem, scheme, N, n, warp, cfl
    ("c1_vortex", "vortex", capi.SCHEME_HYBRIDIZED, 3, 16, 0.0, 0.125),
    ("c2_lake", "lake", capi.SCHEME_HYBRIDIZED, 3, 8, 0.1, 0.125),
    ("dam_n3", "dambreak", capi.SCHEME_HYBRIDIZED, 3, 10, 0.0, 0.0625),
    ("sbp_dam_n4", "dambreak", capi.SCHEME_SBP, 4, 10, 0.0, 0.0625),
    ("sbp_lake_n3", "lake", capi.SCHEME_SBP, 3, 4, 0.1, 0.125),
    ("sbp_vortex_n2", "vortex", capi.SCHEME_SBP, 2, 8, 0.0, 0.125),
]


def eq(a, b):
    np.testing.assert_array_equal(np.asarray(a).reshape(-1), np.asarray(b).reshape(-1))


@pytest.mark.parametrize("name,problem,scheme,N,n,warp,cfl", CASES)
def test_case_matches_reference_bitwise(name, problem, scheme, N, n, warp, cfl):
    g = load_golden(name)
    c = capi.Case(problem, scheme=scheme, N=N, nx=n, warp=warp, cfl=cfl, threads=4)
    assert c.K == int(g["K"][0])
    assert c.dt == float(g["dt"][0])
    assert c.min_edge == float(g["min_edge"][0])
    eq(c.array("map_nodes"), g["map_nodes"])
    eq(c.array("Vq"), g["ref_Vq"])
    eq(c.array("Vf"), g["ref_Vf"])
    eq(c.array("Pq"), g["ref_Pq"])
    eq(c.array("surfq_w"), g["surfq_w"])
    if scheme == capi.SCHEME_SBP:
        eq(c.array("Qr"), g["sbp_Qx"])
        eq(c.array("Qs"), g["sbp_Qy"])
        eq(c.array("M_diag"), g["sbp_M_diag"])
        eq(c.iarray("face_index"), g["sbp_face_index"])
    else:
        eq(c.array("Qr"), g["ref_Qh_x"])
        eq(c.array("Qs"), g["ref_Qh_y"])
        eq(c.array("Mh_inv"), g["Mh_inv"])
    eq(c.array("gf"), g["gf"])
    eq(c.array("J_vol"), g["J_vol"])
    eq(c.array("sJ"), g["sJ"])
    eq(c.array("nx"), g["nx"])
    eq(c.array("ny"), g["ny"])
    eq(c.array("xy_surf"), g["xy_surf"])
    eq(c.iarray("nbr"), g["nbr"])
    eq(c.iarray("nbr_face"), g["nbr_face"])
    eq(c.iarray("face_type"), g["face_type"])
    eq(c.iarray("perm"), g["perm"])
    eq(c.array("face_shift"), g["face_shift"])
    eq(c.u0(), g["u"])
    eq(c.b(), g["b"])


@pytest.mark.parametrize("name,N", [("modal_n4_warp", 4), ("modal_n3_warp", 3), ("modal_n2_walls", 2)])
def test_geometry_of_fixture_meshes(name, N):
    """The test_solver.cpp Fixture meshes ([-1,1]^2, 4x4) — geometry and connectivity."""
    g = load_golden(name)
    warp = 0.1 if "warp" in name else 0.0
    c = capi.Case("lake", N=N, nx=4, warp=warp, threads=2)
    eq(c.array("gf"), g["gf"])
    eq(c.array("Mh_inv"), g["Mh_inv"])
    if "walls" not in name:
        eq(c.iarray("perm"), g["perm"])
        eq(c.iarray("nbr"), g["nbr"])


def test_operator_tables_all_degrees():
    ops = load_golden("ops")
    for N in range(1, 5):
        c = capi.Case("lake", N=N, nx=1, threads=1)
        eq(c.array("Vq"), ops[f"N{N}_Vq"])
        eq(c.array("Pq"), ops[f"N{N}_Pq"])
        eq(c.array("Qr"), ops[f"N{N}_Qh_x"])
        eq(c.array("Qs"), ops[f"N{N}_Qh_y"])
        s = capi.Case("lake", scheme=capi.SCHEME_SBP, N=N, nx=1, threads=1)
        eq(s.array("Qr"), ops[f"N{N}_sbp_Qx"])
        eq(s.array("Qs"), ops[f"N{N}_sbp_Qy"])
        eq(s.iarray("face_index"), ops[f"N{N}_sbp_face_index"])


def test_smooth_workload_is_admissible():
    """The C4/C5 workload generator: smooth_state(seed 23) + lake bathymetry, curved."""
    c = capi.Case("smooth", N=4, nx=32, warp=0.1, threads=4)
    u = c.u0()
    assert u.shape == (2 * 32 * 32, 3, 15)
    assert np.isfinite(u).all()
    assert (c.array("J_vol") > 0).all()
    assert c.dt > 0


def test_invalid_config_raises():
    with pytest.raises(capi.SwedgError):
        capi.Case("lake", N=9, nx=4)
    with pytest.raises(capi.SwedgError):
        capi.Case("lake", N=3, nx=4, cfl=-1.0)
