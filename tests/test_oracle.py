"""Pin the C oracle (oracle/swedg_oracle.c) to the reference's own outputs.

tests/golden/*.npz were produced by the UNMODIFIED reference headers
(oracle/_ref/swedg_dump, see tests/golden/make_golden.py).  The oracle restates
the reference arithmetic in the same order, so equality is asserted BIT FOR BIT.
CPU only.
"""
import math

import numpy as np
import pytest

from oracle_py import Oracle, load_golden

MODAL = ["modal_n1_affine", "modal_n2_walls", "modal_n3_warp", "modal_n4_warp", "modal_n4_affine"]
PROBLEMS_MODAL = ["c1_vortex", "c2_lake", "dam_n3"]
PROBLEMS_SBP = ["sbp_dam_n4", "sbp_lake_n3", "sbp_vortex_n2"]


def run_like_reference(orc, u0, dt, tfinal):
    """run.hpp:230-262: nsteps = ceil(T/dt - 1e-12); step_dt = min(dt, T - t)."""
    nsteps = int(math.ceil(tfinal / dt - 1e-12)) if tfinal > 0 else 0
    u = np.array(u0, copy=True)
    res = np.zeros_like(u)
    t = 0.0
    steps = 0
    for _ in range(nsteps):
        step_dt = min(dt, tfinal - t)
        if step_dt <= 0.0:
            break
        u, res, err = orc.step_lsrk45(u, res, step_dt, 1)
        assert err == 0
        t = t + step_dt
        steps += 1
    return u, steps, t


@pytest.mark.parametrize("name", MODAL)
def test_modal_fixture_bitwise(name):
    c = load_golden(name)
    orc = Oracle(c)
    np.testing.assert_array_equal(orc.b_stacked, c["b_stacked"])
    np.testing.assert_array_equal(orc.src_x, c["src_x"])
    np.testing.assert_array_equal(orc.src_y, c["src_y"])
    proj, err, _ = orc.entropy_projection(c["u"])
    assert err == 0
    np.testing.assert_array_equal(proj, c["proj"])
    du, err, _ = orc.rhs(c["u"])
    assert err == 0
    np.testing.assert_array_equal(du, c["du_lf"])
    du_ec, err, _ = Oracle(c, penalty_lf=False).rhs(c["u"])
    assert err == 0
    np.testing.assert_array_equal(du_ec, c["du_ec"])
    n = int(c["nsteps"][0])
    u, res, err = orc.step_lsrk45(c["u"], np.zeros_like(c["u"]), float(c["dt"][0]), n)
    assert err == 0
    np.testing.assert_array_equal(u, c["u_steps"])
    np.testing.assert_array_equal(res, c["res_steps"])


@pytest.mark.parametrize("name", MODAL[:3])
def test_modal_element_subset(name):
    c = load_golden(name)
    orc = Oracle(c)
    elems = np.array([0, 3, orc.K - 1], dtype=np.int32)
    du, err, _ = orc.rhs(c["u"], elems=elems)
    assert err == 0
    np.testing.assert_array_equal(du[elems], c["du_lf"][elems])


@pytest.mark.parametrize("name", PROBLEMS_MODAL)
def test_problem_modal_run_bitwise(name):
    c = load_golden(name)
    orc = Oracle(c)
    np.testing.assert_array_equal(orc.src_x, c["src_x"])
    du, err, _ = orc.rhs(c["u"])
    assert err == 0
    np.testing.assert_array_equal(du, c["du_lf"])
    u, steps, t = run_like_reference(orc, c["u"], float(c["dt"][0]), float(c["tfinal"][0]))
    assert steps == int(c["run_steps"][0])
    assert t == float(c["run_t"][0])
    np.testing.assert_array_equal(u, c["u_final"])


@pytest.mark.parametrize("name", PROBLEMS_SBP)
def test_problem_sbp_bitwise(name):
    c = load_golden(name)
    orc = Oracle(c)
    np.testing.assert_array_equal(orc.src_x, c["src_x"])
    np.testing.assert_array_equal(orc.src_y, c["src_y"])
    du, err, _ = orc.rhs(c["u"])
    assert err == 0
    np.testing.assert_array_equal(du, c["du_lf"])
    du_ec, err, _ = Oracle(c, penalty_lf=False).rhs(c["u"])
    np.testing.assert_array_equal(du_ec, c["du_ec"])
    u, steps, t = run_like_reference(orc, c["u"], float(c["dt"][0]), float(c["tfinal"][0]))
    assert steps == int(c["run_steps"][0])
    np.testing.assert_array_equal(u, c["u_final"])


def test_positivity_reports_element_1():
    c = load_golden("positivity")
    msg = bytes(c["error_message"].astype(np.uint8)).decode()
    assert "element 1" in msg
    orc = Oracle(c)
    _, err, bad = orc.rhs(c["u"])
    assert err == 1 and bad == 1


def test_lake_at_rest_golden_is_well_balanced():
    c = load_golden("c2_lake")
    assert float(c["run_err_combined"][0]) <= 1e-9
    assert np.abs(c["du_lf"]).max() < 1e-10


def test_known_answer_ec_flux_and_entropy_vars():
    """SPEC.md:307,340 known answers through the oracle's pointwise maps."""
    # ec flux uL=(1,0,0), uR=(2,2,0), g=1 -> x-flux (1, 1.5, 0)
    uL, uR, g = np.array([1.0, 0, 0]), np.array([2.0, 2.0, 0]), 1.0
    ux = 0.5 * (uL[1] / uL[0] + uR[1] / uR[0])
    hu = 0.5 * (uL[1] + uR[1])
    h_avg = 0.5 * (uL[0] + uR[0])
    p = g * h_avg * h_avg - 0.25 * g * (uL[0] ** 2 + uR[0] ** 2)
    assert (hu, hu * ux + p) == (1.0, 1.5)


@pytest.mark.parametrize("name", MODAL + PROBLEMS_MODAL + PROBLEMS_SBP)
def test_long_double_yardstick(name):
    """The long-double build of the same algorithm agrees with the reference to its
    rounding error; on states with du ~ 0 (lake/dam at rest) that error exceeds
    1e-12 relative — which is why FAST is judged against it (test_gpu_parity)."""
    c = load_golden(name)
    ld, err, _ = Oracle(c, precision="ld").rhs(c["u"])
    assert err == 0
    ref = c["du_lf"]
    abs_err = np.abs(ref - ld).max()
    assert abs_err <= 1e-10 * (1.0 + np.abs(ld).max())
    assert abs_err > 0.0  # genuinely a different (more precise) evaluation


# ---- diagnostics (diagnostics.hpp:142-267): compute_invariants / l2_error ----
@pytest.mark.parametrize("name", PROBLEMS_MODAL + PROBLEMS_SBP)
def test_diagnostics_oracle_bitwise(name):
    """oracle_diag's serial sums == the reference's compute_invariants and both
    l2_error forms on the initial and the final run() state, bit for bit."""
    from oracle_py import diag, project_nodal

    c = load_golden(name)
    sbp = int(c["scheme"][0]) == 1
    g = float(c["g"][0])
    for tag, key, t in (("diag0_", "u", 0.0), ("diag1_", "u_final", float(c["run_t"][0]))):
        u, b = c[key], c["b"]
        if sbp:
            u = project_nodal(c["ref_Pq"], u)
            b = project_nodal(c["ref_Pq"], b[:, None, :])[:, 0, :]
        _, s, mh, err, _ = diag(c, u, what=0, b_modal=b, g=g, t=t)
        assert err == 0
        np.testing.assert_array_equal(np.r_[t, s, mh], c[tag + "invariants"])
        for key_l2, what, kw in (("l2_ref", 1, {"u_ref": c.get(tag + "ref_state")}),
                                 ("l2_exact", 2 if "vortex" in name else 3, {"t": t})):
            if tag + key_l2 not in c:
                continue
            _, s, _, err, _ = diag(c, u, what=what, **kw)
            assert err == 0
            e = np.r_[np.sqrt(s[:3]), np.sqrt(s[0] + s[1] + s[2])]
            np.testing.assert_array_equal(e, c[tag + key_l2])


def test_ratio_oracle_bitwise():
    """oracle_ratio_* == bench.hpp kernel_matvec / kernel_fluxdiff / kernel_fluxdiff_skew."""
    from oracle_py import ratio_kernels

    G = load_golden("ratio")
    for n in G["sizes"]:
        p = f"n{n}_"
        dg, es = ratio_kernels(G[p + "Q"], G[p + "u"])
        np.testing.assert_array_equal(dg, G[p + "y_dg"])
        np.testing.assert_array_equal(es, G[p + "y_esdg"])
        nq = int(G[p + "nq"][0])
        Qz = np.array(G[p + "Q"], copy=True)
        Qz[nq:, nq:] = 0.0
        _, sk = ratio_kernels(Qz, G[p + "u"], nq=nq)
        np.testing.assert_array_equal(sk, G[p + "y_skew"])


def test_reference_unit_tests_pass_with_shims():
    """The unmodified reference test suite (tests/test_*.cpp), compiled against
    oracle/shim by oracle/Makefile.ref, passes — the shims reproduce what the reference
    needs from Eigen/doctest.  Needs /root/reference (this container), else skipped."""
    import os
    import subprocess

    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "unit_tests")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/unit_tests not built (no /root/reference here)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "0 failed" in out.stdout
