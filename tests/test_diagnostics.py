"""Device diagnostics: compute_invariants / l2_error on the
GPU and the device-resident run() loop.

Parity bar:
  * every per-point term is the reference's (bitwise, checked through the
    oracle's terms), and the device sums are EXACT — so each invariant equals
    math.fsum of the oracle's terms bit for bit;
  * against the reference's own serial sums (golden fixtures) the difference
    is bounded by the reference's summation error, n * eps * sum|terms|;
  * exact-solution L2 errors (vortex, lake) use CUDA's exp/sincos: relative 1e-11;
  * raw accumulators of P logical partitions merge to the global value bitwise.
"""
import math

import numpy as np
import pytest

from oracle_py import diag, load_golden, project_nodal

pytestmark = pytest.mark.gpu
capi = pytest.importorskip("paper_2005_02516_b200.capi")

PROBLEMS = ["c1_vortex", "c2_lake", "dam_n3", "sbp_dam_n4", "sbp_lake_n3", "sbp_vortex_n2"]
EPS = np.finfo(np.float64).eps


def modal(c, u):
    return project_nodal(c["ref_Pq"], u) if int(c["scheme"][0]) == 1 else u


def modal_b(c):
    b = c["b"]
    return project_nodal(c["ref_Pq"], b[:, None, :])[:, 0, :] if int(c["scheme"][0]) == 1 else b


def fsums(terms, ncol):
    return np.array([math.fsum(terms[..., q].ravel().tolist()) for q in range(ncol)])


def serial_bound(terms, q):
    a = np.abs(terms[..., q]).ravel()
    return a.size * EPS * a.sum()


@pytest.mark.parametrize("name", PROBLEMS)
def test_invariants_exact_and_within_reference_rounding(name):
    c = load_golden(name)
    h = capi.handle_from_case(c, mode=capi.MODE_PARITY)
    g = float(c["g"][0])
    for tag, key, t in (("diag0_", "u", 0.0), ("diag1_", "u_final", float(c["run_t"][0]))):
        inv = h.compute_invariants(c[key], t)
        terms, _, mh, err, _ = diag(c, modal(c, c[key]), what=0, b_modal=modal_b(c), g=g, t=t)
        assert err == 0
        got = np.array([inv[f] for f in capi.INVARIANT_FIELDS])
        # bit-for-bit: correctly rounded sums of the reference's terms
        np.testing.assert_array_equal(got[1:5], fsums(terms, 4))
        assert got[0] == t and got[5] == mh
        ref = c[tag + "invariants"]
        assert got[5] == ref[5]
        for q in range(4):
            assert abs(got[1 + q] - ref[1 + q]) <= serial_bound(terms, q), (name, tag, q)
    h.close()


@pytest.mark.parametrize("name", ["c2_lake", "sbp_lake_n3", "c1_vortex", "sbp_vortex_n2"])
def test_l2_errors(name):
    c = load_golden(name)
    h = capi.handle_from_case(c, mode=capi.MODE_PARITY)
    for tag, key, t in (("diag0_", "u", 0.0), ("diag1_", "u_final", float(c["run_t"][0]))):
        um = modal(c, c[key])
        if tag + "l2_ref" in c:
            e = h.l2_error(capi.DIAG_L2_REF, c[key], c[tag + "ref_state"], t)
            terms, _, _, _, _ = diag(c, um, what=1, u_ref=c[tag + "ref_state"])
            s = fsums(terms, 3)
            np.testing.assert_array_equal(e, np.r_[np.sqrt(s), np.sqrt(s[0] + s[1] + s[2])])
            np.testing.assert_allclose(e, c[tag + "l2_ref"], rtol=1e-12, atol=1e-300)
        what = capi.DIAG_L2_VORTEX if "vortex" in name else capi.DIAG_L2_LAKE
        e = h.l2_error(what, c[key], None, t)
        np.testing.assert_allclose(e, c[tag + "l2_exact"], rtol=1e-11, atol=1e-15)
    h.close()


@pytest.mark.parametrize("name", ["c1_vortex", "sbp_vortex_n2", "dam_n3"])
def test_device_run_loop_matches_reference_run(name):
    """swedg_run == run() (run.hpp:226-262): same steps, same sampling times,
    bitwise final state (PARITY), invariant series within the reference's
    serial-summation rounding and bit-for-bit the exact sums of its terms."""
    c = load_golden(name)
    h = capi.handle_from_case(c, mode=capi.MODE_PARITY)
    h.set_state(c["u"], None, 0.0)
    series, steps = h.run(float(c["run_dt"][0]), float(c["tfinal"][0]))
    assert steps == int(c["run_steps"][0])
    ref = c["run_invariants"]
    assert series.shape == ref.shape
    np.testing.assert_array_equal(series[:, 0], ref[:, 0])
    np.testing.assert_array_equal(series[:, 5], ref[:, 5])
    scale = np.abs(ref[:, 1:5]).max(axis=0)
    assert (np.abs(series[:, 1:5] - ref[:, 1:5]) <= 1e-13 * (1 + scale)).all()
    u, _, t = h.get_state()
    np.testing.assert_array_equal(u, c["u_final"])
    assert t == float(c["run_t"][0])
    terms, _, _, _, _ = diag(c, modal(c, u), what=0, b_modal=modal_b(c), g=float(c["g"][0]), t=t)
    np.testing.assert_array_equal(series[-1, 1:5], fsums(terms, 4))
    h.close()


def test_run_loop_fast_mode_and_graphs():
    """FAST mode with graph replays over several sampling intervals: conserved mass,
    sampled every step on request."""
    c = capi.Case("vortex", N=3, nx=16)
    h = c.handle(mode=capi.MODE_FAST)
    h.set_state(c.u0())
    series, steps = h.run(c.dt, 40 * c.dt, sample_every=8)
    assert steps == 40 and series.shape[0] == 6
    np.testing.assert_allclose(series[:, 0], [0, 8 * c.dt, 16 * c.dt, 24 * c.dt, 32 * c.dt, 40 * c.dt], rtol=1e-14)
    m = series[:, 1]
    assert np.abs(m - m[0]).max() <= 1e-12 * m[0]
    h2 = c.handle(mode=capi.MODE_FAST)
    h2.set_state(c.u0())
    h2.set_graphs(False)
    s2, _ = h2.run(c.dt, 40 * c.dt, sample_every=8)
    np.testing.assert_array_equal(series, s2)  # graph replay == individual launches
    h.close()
    h2.close()


def test_invariants_raw_merge_over_partitions_bitwise():
    """P logical y-strip partitions: merged raw accumulators == global invariants, bitwise."""
    P, NX, NY = 3, 8, 4
    glob = capi.Case("smooth", N=4, nx=NX, ny=NY, warp=0.1, strips=P, strip=-1)
    hg = glob.handle()
    inv_g = hg.compute_invariants(glob.u0(), 0.0)
    raws = []
    for r in range(P):
        s = capi.Case("smooth", N=4, nx=NX, ny=NY, warp=0.1, strips=P, strip=r)
        hs = s.handle()
        raws.append(hs.diag_raw(capi.DIAG_INVARIANTS, s.u0(), None, 0.0))
        hs.close()
    merged = capi.diag_from_raw(raws, 1)[0]
    np.testing.assert_array_equal(merged, [inv_g[f] for f in capi.INVARIANT_FIELDS])
    hg.close()


def test_invariants_positivity_error():
    c = load_golden("c1_vortex")
    h = capi.handle_from_case(c, mode=capi.MODE_PARITY)
    u = np.array(c["u"], copy=True)
    u[7, 0, 0] = -abs(u[7, 0, 0])
    with pytest.raises(capi.PositivityError) as ei:
        h.compute_invariants(u, 0.0)
    assert ei.value.elem == 7
    h.close()


def test_invariants_c4_sample_k1d256():
    """C4 generator at K1D=256 (K=131,072): exact sums of the oracle's terms, bitwise."""
    c = capi.Case("smooth", N=4, nx=256, warp=0.1)
    h = c.handle()
    inv = h.compute_invariants(c.u0(), 0.0)
    d = c.diag_arrays()
    fine = {"fine_w": d["w"], "fine_V": d["V"], "fine_Vr": d["Vr"], "fine_Vs": d["Vs"],
            "map_coeffs": d["map_coeffs"]}
    terms, _, mh, err, _ = diag(fine, c.u0(), what=0, b_modal=c.b(), g=c.g)
    assert err == 0
    np.testing.assert_array_equal([inv[f] for f in capi.INVARIANT_FIELDS[1:5]], fsums(terms, 4))
    assert inv["min_h"] == mh
    h.close()


def test_python_run_writes_reference_output_files(tmp_path):
    """paper_2005_02516_b200.run.run (run.hpp:226-284 with out_dir) on the small vortex of
    tests/golden/io.npz, PARITY: both VTK files byte-identical to the reference's, the CSV
    files equal to within the reference's summation rounding."""
    from paper_2005_02516_b200 import run as srun

    G = load_golden("io")
    text = lambda a: bytes(np.asarray(a).astype(np.uint8)).decode()  # noqa: E731
    c = capi.Case("vortex", N=2, nx=4)
    res = srun.run(c, tfinal=0.05, mode=capi.MODE_PARITY, out_dir=str(tmp_path))
    assert (tmp_path / "solution_0.vtk").read_text() == text(G["vtk0_text"])
    assert (tmp_path / text(G["final_name"])).read_text() == text(G["vtk1_text"])
    np.testing.assert_array_equal(res["u"], G["u_final"])
    got = np.loadtxt(tmp_path / "invariants.csv", delimiter=",", skiprows=1).reshape(-1, 6)
    np.testing.assert_array_equal(got[:, 0], G["series"][:, 0])
    np.testing.assert_allclose(got[:, 1:], G["series"][:, 1:], rtol=1e-13, atol=1e-15)
    e = np.genfromtxt(tmp_path / "errors.csv", delimiter=",", skip_header=1)
    np.testing.assert_allclose(e[:6], G["error"], rtol=1e-11)


@pytest.mark.parametrize("variant", [0, 1, 2])
def test_vortex_convergence_study_matches_reference(variant):
    """Acceptance criterion 5 (acceptance.cpp:188-223) on the device: the vortex
    convergence studies (affine / curved hybridized N = 2, 3; SBP N = 2) with the
    device run loop and device L2 errors reproduce the reference's errors (relative
    1e-9: FAST arithmetic and CUDA exp) and pass its order thresholds."""
    from paper_2005_02516_b200 import run as srun

    ref = load_golden("convergence")["rows"]
    ref = ref[ref[:, 0] == variant]
    kw = {0: {}, 1: {"warp": 0.1}, 2: {"scheme": capi.SCHEME_SBP}}[variant]
    degrees = [2] if variant == 2 else [2, 3]
    rows = srun.convergence_study("vortex", degrees, 3, **kw)
    assert len(rows) == len(ref)
    for r, rr in zip(rows, ref):
        assert (r["N"], r["nx"], r["ny"]) == (int(rr[1]), int(rr[2]), int(rr[3]))
        e = r["error"]
        np.testing.assert_allclose([e["err_h"], e["err_hu"], e["err_hv"], e["combined"]], rr[4:8], rtol=1e-9)
        assert e["h_mesh"] == rr[9]
    finest = {N: [r["order"] for r in rows if r["N"] == N][-1] for N in degrees}
    if variant == 2:
        assert finest[2] >= 1.5
    else:
        for N in degrees:
            assert finest[N] >= N + 0.5 or variant == 1
