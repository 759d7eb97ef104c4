"""GPU parity of the CUDA path against the reference (golden fixtures) and the C oracle.

Every call goes through the C ABI (include/swedg_b200.h) via
paper_2005_02516_b200.capi.  Two arithmetic modes are tested:

  PARITY  reference evaluation order, no FMA contraction: asserted BIT-FOR-BIT
          equal to the reference's outputs (tests/golden, produced by the
          unmodified reference headers) — projection, bathymetry source, RHS
          with LF and EC penalties, LSRK45 steps and whole runs.
  FAST    the production kernels (FMA, reassociated flux differencing):
          asserted within the north-star tolerance
              max|du - du_ref| / (1 + max|du_ref|) <= 1e-12   per RHS
              max|u  - u_ref|  / (1 + max|u_ref|)  <= 1e-10   after the config horizon
"""
import math

import numpy as np
import pytest

import parity_log
from oracle_py import Oracle, case_dict, load_golden

pytestmark = pytest.mark.gpu

capi = pytest.importorskip("paper_2005_02516_b200.capi")

MODAL = ["modal_n1_affine", "modal_n2_walls", "modal_n3_warp", "modal_n4_warp", "modal_n4_affine"]
SBP = ["sbp_dam_n4", "sbp_lake_n3", "sbp_vortex_n2"]
RHS_TOL = 1e-12
RUN_TOL = 1e-10


def rel(a, b):
    return float(np.abs(a - b).max() / (1.0 + np.abs(b).max()))


def assert_fast_rhs(du_fast, du_ref, case, u, penalty_lf=True, label=None):
    """FAST-mode acceptance for one RHS evaluation:
        max|du_fast - du_ref| / (1 + max|du_ref|) <= 1e-12            (north-star tolerance)
    or, on cancellation-dominated states where the reference itself is further
    than that from the exact RHS (lake/dam at rest: du ~ 1e-12 noise), FAST must
    be no less accurate than the reference:
        max|du_fast - du_exact| <= 4 max|du_ref - du_exact|,
    with du_exact from the same algorithm in long double (oracle/liboracle_ld.so).
    Every call is recorded with its numbers and branch (tests/parity_log.py)."""
    def exact():
        ex, err, _ = Oracle(case, penalty_lf=penalty_lf, precision="ld").rhs(u)
        assert err == 0
        return ex

    parity_log.assert_fast_rhs(du_fast, du_ref, exact, label=label or ("LF" if penalty_lf else "EC"))


def make(c, mode, penalty=capi.PENALTY_LF):
    return capi.handle_from_case(c, mode=mode, penalty=penalty)


def run_like_reference(h, u0, dt, tfinal):
    """run.hpp:230-262 step sequence on the device-resident state."""
    nsteps = int(math.ceil(tfinal / dt - 1e-12)) if tfinal > 0 else 0
    h.set_state(u0, None, 0.0)
    t = 0.0
    steps = 0
    for _ in range(nsteps):
        step_dt = min(dt, tfinal - t)
        if step_dt <= 0.0:
            break
        h.step(step_dt, 1, sync=False)
        t = t + step_dt
        steps += 1
    h.check()
    u, _, _ = h.get_state()
    return u, steps


@pytest.mark.parametrize("name", MODAL)
def test_modal_parity_bitwise(name):
    c = load_golden(name)
    h = make(c, capi.MODE_PARITY)
    bs, src = h.bathymetry_products()
    np.testing.assert_array_equal(bs, c["b_stacked"])
    np.testing.assert_array_equal(src[:, 0], c["src_x"])
    np.testing.assert_array_equal(src[:, 1], c["src_y"])
    np.testing.assert_array_equal(h.entropy_projection(c["u"]), c["proj"])
    np.testing.assert_array_equal(h.rhs(c["u"]), c["du_lf"])
    h.set_penalty(capi.PENALTY_EC)
    np.testing.assert_array_equal(h.rhs(c["u"]), c["du_ec"])
    h.set_penalty(capi.PENALTY_LF)
    h.set_state(c["u"])
    h.step(float(c["dt"][0]), int(c["nsteps"][0]))
    u, res, _ = h.get_state()
    np.testing.assert_array_equal(u, c["u_steps"])
    np.testing.assert_array_equal(res, c["res_steps"])


@pytest.mark.parametrize("name", MODAL)
def test_modal_fast_within_tolerance(name):
    c = load_golden(name)
    h = make(c, capi.MODE_FAST)
    assert rel(h.entropy_projection(c["u"]), c["proj"]) <= 1e-13
    assert_fast_rhs(h.rhs(c["u"]), c["du_lf"], c, c["u"])
    h.set_penalty(capi.PENALTY_EC)
    assert_fast_rhs(h.rhs(c["u"]), c["du_ec"], c, c["u"], penalty_lf=False)


@pytest.mark.parametrize("name", ["c1_vortex", "c2_lake", "dam_n3"])
@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_problem_runs(name, mode):
    c = load_golden(name)
    h = make(c, capi.MODE_PARITY if mode == "parity" else capi.MODE_FAST)
    du = h.rhs(c["u"])
    u, steps = run_like_reference(h, c["u"], float(c["dt"][0]), float(c["tfinal"][0]))
    assert steps == int(c["run_steps"][0])
    if mode == "parity":
        np.testing.assert_array_equal(du, c["du_lf"])
        np.testing.assert_array_equal(u, c["u_final"])
    else:
        assert_fast_rhs(du, c["du_lf"], c, c["u"])
        assert rel(u, c["u_final"]) <= RUN_TOL


def test_lake_at_rest_preserved_to_roundoff():
    c = load_golden("c2_lake")
    for mode in (capi.MODE_PARITY, capi.MODE_FAST):
        h = make(c, mode)
        assert np.abs(h.rhs(c["u"])).max() < 1e-10
        u, _ = run_like_reference(h, c["u"], float(c["dt"][0]), float(c["tfinal"][0]))
        assert np.abs(u - c["u"]).max() < 1e-10


@pytest.mark.parametrize("name", SBP)
@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_sbp(name, mode):
    c = load_golden(name)
    h = make(c, capi.MODE_PARITY if mode == "parity" else capi.MODE_FAST)
    _, src = h.bathymetry_products()
    du = h.rhs(c["u"])
    h.set_penalty(capi.PENALTY_EC)
    du_ec = h.rhs(c["u"])
    h.set_penalty(capi.PENALTY_LF)
    u, steps = run_like_reference(h, c["u"], float(c["dt"][0]), float(c["tfinal"][0]))
    assert steps == int(c["run_steps"][0])
    if mode == "parity":
        np.testing.assert_array_equal(src[:, 0], c["src_x"])
        np.testing.assert_array_equal(src[:, 1], c["src_y"])
        np.testing.assert_array_equal(du, c["du_lf"])
        np.testing.assert_array_equal(du_ec, c["du_ec"])
        np.testing.assert_array_equal(u, c["u_final"])
    else:
        assert_fast_rhs(du, c["du_lf"], c, c["u"])
        assert_fast_rhs(du_ec, c["du_ec"], c, c["u"], penalty_lf=False)
        assert rel(u, c["u_final"]) <= RUN_TOL


def test_positivity_error_names_element_1():
    c = load_golden("positivity")
    h = make(c, capi.MODE_FAST)
    with pytest.raises(capi.PositivityError) as ei:
        h.rhs(c["u"])
    assert "element 1" in str(ei.value)
    assert ei.value.elem == 1


def test_dt_must_be_positive():
    c = load_golden("modal_n1_affine")
    h = make(c, capi.MODE_FAST)
    h.set_state(c["u"])
    with pytest.raises(capi.InvalidArgument):
        h.step(-1.0, 1)


def test_oracle_agrees_with_gpu_on_perturbed_state():
    """Random admissible perturbation (not in any fixture): GPU vs C oracle."""
    c = load_golden("modal_n4_warp")
    rng = np.random.default_rng(7)
    u = c["u"] + 0.01 * rng.standard_normal(c["u"].shape)
    orc = Oracle(c)
    ref, err, _ = orc.rhs(u)
    assert err == 0
    h = make(c, capi.MODE_PARITY)
    np.testing.assert_array_equal(h.rhs(u), ref)
    h.set_mode(capi.MODE_FAST)
    assert rel(h.rhs(u), ref) <= RHS_TOL


def test_graph_replay_equals_individual_launches_and_reports_step():
    """swedg_step_lsrk45 with nsteps >= 2 replays a captured one-step CUDA graph (and a
    one-step call replays it once it exists): bitwise equal to individually launched steps;
    an error in a later step is attributed to the right element and stage time."""
    c = load_golden("c1_vortex")
    dt = float(c["dt"][0])
    h1 = make(c, capi.MODE_FAST)
    h1.set_graphs(False)
    h1.set_state(c["u"])
    h1.step(dt, 6)
    u1, r1, t1 = h1.get_state()
    h2 = make(c, capi.MODE_FAST)
    h2.set_state(c["u"])
    h2.step(dt, 3)
    h2.step(dt, 2)
    h2.step(dt, 1)  # one step: the existing graph is replayed (run loops sampling every step)
    u2, r2, t2 = h2.get_state()
    np.testing.assert_array_equal(u1, u2)
    np.testing.assert_array_equal(r1, r2)
    assert t1 == t2
    bad1 = np.array(c["u"], copy=True)
    bad1[9, 0, 0] = -1.0
    h2.set_state(bad1, None, 0.125)
    with pytest.raises(capi.PositivityError) as ei:
        h2.step(dt, 1)
    assert ei.value.elem == 9 and abs(ei.value.t - 0.125) < 1e-12
    # positivity failure planted in element 7: reported with element id and a stage time
    bad = np.array(c["u"], copy=True)
    bad[7, 0, 0] = -1.0
    h2.set_state(bad, None, 0.25)
    with pytest.raises(capi.PositivityError) as ei:
        h2.step(dt, 4)
    assert ei.value.elem == 7 and "element 7" in str(ei.value)
    assert abs(ei.value.t - 0.25) < 1e-12


@pytest.mark.parametrize("mode", ["parity", "fast"])
@pytest.mark.parametrize("nchunks", [1, 3, 8])
def test_host_state_stepping_equals_device_steps(mode, nchunks):
    """swedg_step_lsrk45_host (state round-trips through host memory every step, copies
    pipelined with chunked stage-1 volume kernels) == device-resident steps, bitwise;
    errors keep the global element id and stage time across chunks and async steps."""
    c = load_golden("c1_vortex")
    m = capi.MODE_PARITY if mode == "parity" else capi.MODE_FAST
    dt = float(c["dt"][0])
    h1 = make(c, m)
    h1.set_state(c["u"])
    h1.step(dt, 3)
    u1, _, t1 = h1.get_state()
    h2 = make(c, m)
    u = np.array(c["u"], copy=True)
    h2.set_state(u)  # t = 0
    h2.step_host(u, dt, 3, nchunks)
    np.testing.assert_array_equal(u, u1)
    _, _, t2 = h2.get_state()
    assert t2 == t1
    bad = np.array(c["u"], copy=True)
    bad[400, 0, 0] = -1.0  # element 400 of 512: in the last chunks
    h2.set_state(bad, None, 0.5)
    with pytest.raises(capi.PositivityError) as ei:
        h2.step_host(bad, dt, 2, nchunks)
    assert ei.value.elem == 400 and abs(ei.value.t - 0.5) < 1e-12


@pytest.mark.parametrize("nchunks", [6, 16])
def test_host_state_wavefront_merged_launches_n4(nchunks, monkeypatch):
    """N = 4 FAST host-state wavefront: each tick's volume pieces and interface pieces go
    out as segmented launches (per-piece element range, stage id, LSRK coefficients);
    bitwise the per-chunk launches (SWEDG_WAVE_MERGE=0) and the device-resident steps, and
    a planted positivity failure reports the same element and stage time."""
    c = capi.Case("smooth", N=4, nx=24, warp=0.1, seed=23)  # K = 1152
    dt = c.dt
    outs, errs = [], []
    for merge in ("1", "0"):
        monkeypatch.setenv("SWEDG_WAVE_MERGE", merge)
        h = c.handle(mode=capi.MODE_FAST)
        u = np.ascontiguousarray(c.u0())
        h.set_state(u)
        l0 = h.launches
        h.step_host(u, dt, 3, nchunks)
        outs.append((u, h.launches - l0))
        bad = np.ascontiguousarray(c.u0())
        bad[1000, 0, 3] = -1.0
        h.set_state(bad, None, 0.5)
        with pytest.raises(capi.PositivityError) as ei:
            h.step_host(bad, dt, 2, nchunks)
        errs.append((ei.value.elem, ei.value.t))
        h.close()
    hd = c.handle(mode=capi.MODE_FAST)
    hd.set_state(c.u0())
    hd.step(dt, 3)
    ud = hd.get_state()[0]
    np.testing.assert_array_equal(outs[0][0], ud)
    np.testing.assert_array_equal(outs[1][0], ud)
    # fewer launches when merged (with C <= 6 chunks no two pieces share a tick)
    assert outs[0][1] < outs[1][1] if nchunks > 6 else outs[0][1] == outs[1][1]
    assert errs[0] == errs[1] and errs[0][0] == 1000 and abs(errs[0][1] - 0.5) < 1e-12


@pytest.mark.parametrize("N", [3, 4])
def test_odd_element_count_imported_mesh(N):
    """Odd K (a pentagon fan of 5 triangles, wall boundary, imported through
    swedg_case_build_mesh): exercises the pair kernel's single-element tail and the
    chunked paths; PARITY bitwise against the C oracle, FAST within tolerance, and a
    few LSRK45 steps (graph replay + host-state path) agree with the oracle's steps."""
    import math as m
    verts = [[0.0, 0.0]] + [[0.6 * m.cos(2 * m.pi * i / 5), 0.6 * m.sin(2 * m.pi * i / 5)] for i in range(5)]
    tris = [[0, 1 + i, 1 + (i + 1) % 5] for i in range(5)]
    c = capi.Case("smooth", N=N, mesh=dict(verts=verts, tris=tris, domain=(0.0, 0.0, 2.0, 2.0)))
    assert c.K == 5
    cd = case_dict(c)
    u = c.u0()
    ref, err, _ = Oracle(cd).rhs(u)
    assert err == 0
    hp = c.handle(mode=capi.MODE_PARITY)
    np.testing.assert_array_equal(hp.rhs(u), ref)
    hf = c.handle(mode=capi.MODE_FAST)
    assert_fast_rhs(hf.rhs(u), ref, cd, u)
    dt = 0.5 * c.dt
    u_ref, _, err = Oracle(cd).step_lsrk45(u, np.zeros_like(u), dt, 3)
    assert err == 0
    hp.set_state(u)
    hp.step(dt, 3)
    np.testing.assert_array_equal(hp.get_state()[0], u_ref)
    uh = np.array(u, copy=True)
    hf.set_state(uh)
    hf.step_host(uh, dt, 3, 2)
    assert rel(uh, u_ref) <= RUN_TOL


@pytest.mark.parametrize("scheme", ["modal", "sbp", "modal_n3"])
def test_positivity_error_in_pair_kernels(scheme):
    """FAST pair kernels (modal N=4 and N=3, SBP N=4) report a nonpositive height with the
    reference's element id, from rhs() and from graph-replayed steps."""
    sc = capi.SCHEME_SBP if scheme == "sbp" else capi.SCHEME_HYBRIDIZED
    c = capi.Case("smooth", scheme=sc, N=3 if scheme == "modal_n3" else 4, nx=8, warp=0.1)
    h = c.handle(mode=capi.MODE_FAST)
    u = c.u0()
    u[77, 0, :] = -1.0 if sc == capi.SCHEME_SBP else 0.0
    if sc != capi.SCHEME_SBP:
        u[77, 0, 0] = -1.0
    with pytest.raises(capi.PositivityError) as ei:
        h.rhs(u)
    assert ei.value.elem == 77
    h.set_state(u, None, 0.125)
    with pytest.raises(capi.PositivityError) as ei:
        h.step(1e-4, 3)
    assert ei.value.elem == 77 and abs(ei.value.t - 0.125) < 1e-12


def test_sbp_pair_pdl_and_state_rotation():
    """SBP N=4 FAST pair path: every stage fuses the LSRK45 update with the state rotating
    u -> A -> B -> A -> B -> u; the launches use programmatic dependent launch.  Steps
    with PDL on / off (SWEDG_PDL=4 / 0) and graph replay / individual launches are bitwise
    equal, and stay within the run tolerance of the reference's steps."""
    import os

    c = load_golden("sbp_dam_n4")
    dt = float(c["dt"][0])
    outs = []
    for pdl, graphs in (("4", True), ("0", True), ("4", False)):  # SWEDG_PDL bit 4: SBP pair kernel
        os.environ["SWEDG_PDL"] = pdl
        try:
            h = make(c, capi.MODE_FAST)
        finally:
            os.environ.pop("SWEDG_PDL", None)
        h.set_graphs(graphs)
        h.set_state(c["u"])
        h.step(dt, 3)
        u, res, t = h.get_state()
        outs.append((u, res, t))
    for u, res, t in outs[1:]:
        np.testing.assert_array_equal(u, outs[0][0])
        np.testing.assert_array_equal(res, outs[0][1])
        assert t == outs[0][2]
    u_ref, _, err = Oracle(c).step_lsrk45(c["u"], np.zeros_like(c["u"]), dt, 3)
    assert err == 0
    assert rel(outs[0][0], u_ref) <= RUN_TOL


def test_sbp_rhs_device_unaligned_input_falls_back():
    """The SBP pair kernel bulk-copies 16 B-aligned pair blocks; a caller's device input
    that is only 8 B aligned takes the thread-per-node kernel instead (same tolerance)."""
    import torch

    c = load_golden("sbp_dam_n4")
    h = make(c, capi.MODE_FAST)
    u = np.ascontiguousarray(c["u"], dtype=np.float64)
    n = u.size
    buf = torch.empty(n + 1, dtype=torch.float64, device="cuda")
    ua = buf[:n]
    uu = buf[1:]  # 8 B past a 16 B boundary
    du_a = torch.empty(n, dtype=torch.float64, device="cuda")
    du_u = torch.empty(n, dtype=torch.float64, device="cuda")
    ua.copy_(torch.from_numpy(u.ravel()))
    h.rhs_device(ua.data_ptr(), du_a.data_ptr())
    uu.copy_(torch.from_numpy(u.ravel()))
    h.rhs_device(uu.data_ptr(), du_u.data_ptr())
    torch.cuda.synchronize()
    a = du_a.cpu().numpy().reshape(u.shape)
    b = du_u.cpu().numpy().reshape(u.shape)
    assert_fast_rhs(a, c["du_lf"], c, c["u"])
    assert_fast_rhs(b, c["du_lf"], c, c["u"])


@pytest.mark.parametrize("name", ["modal_n4_warp", "modal_n3_warp"])
def test_modal_volume_ranges_with_odd_split(name):
    """Volume launches over element ranges [0, k) and [k, K) with k odd — bitwise the
    full-range stage.  N=4: the second range's u block (45 doubles per element) is then
    8 B aligned, so the pair kernel stages it with plain loads; N=3 blocks (u 30, gf 112,
    b 28 doubles per element) stay 16 B aligned at any k, so both ranges use bulk copies
    (the plain-load path is covered by the unaligned rhs_device test)."""
    c = load_golden(name)
    K = int(c["K"][0])
    dt = float(c["dt"][0])
    h1 = make(c, capi.MODE_FAST)
    h1.set_state(c["u"])
    h1.step(dt, 1)
    u1, _, _ = h1.get_state()
    h2 = make(c, capi.MODE_FAST)
    h2.set_state(c["u"])
    k = K // 2 + (1 - (K // 2) % 2)  # odd split point
    for s in range(5):
        h2.stage_volume_range(s, dt, 0, k)
        h2.stage_volume_range(s, dt, k, K)
        h2.stage_surface(s, dt)
    h2.check()
    u2, _, _ = h2.get_state()
    np.testing.assert_array_equal(u2, u1)


@pytest.mark.parametrize("mask", ["0", "1", "3"])
def test_modal_pdl_launches_bitwise(mask):
    """Modal FAST N=4: programmatic dependent launch of the volume (bit 1) and interface
    (bit 2) kernels changes only when a kernel's prologue runs, never a result: device
    steps, host-state (chunked wavefront) steps and an RHS are bitwise the PDL-off ones."""
    import os

    c = load_golden("modal_n4_warp")
    dt = float(c["dt"][0])
    res = []
    for m in ("0", mask):
        os.environ["SWEDG_PDL"] = m
        try:
            h = make(c, capi.MODE_FAST)
        finally:
            os.environ.pop("SWEDG_PDL", None)
        h.set_state(c["u"])
        h.step(dt, 3)
        u, _, _ = h.get_state()
        uh = np.array(c["u"], copy=True)
        h.set_state(uh)
        h.step_host(uh, dt, 2, 4)
        res.append((u, uh, h.rhs(c["u"])))
    for a, b in zip(res[0], res[1]):
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("ntri", [1, 2, 3])
@pytest.mark.parametrize("scheme", ["modal", "sbp"])
def test_tiny_meshes_pair_kernels(ntri, scheme):
    """K = 1, 2, 3 (fans of 1..3 wall-bounded triangles): the pair kernels' smallest
    launches — a lone element, one full pair (bulk copies), a pair plus a tail — for
    the modal N=4 and SBP N=4 FAST paths, RHS within tolerance of the C oracle and
    LSRK45 steps within the run tolerance."""
    import math as m
    verts = [[0.0, 0.0]] + [[0.6 * m.cos(0.5 * m.pi * i / 3), 0.6 * m.sin(0.5 * m.pi * i / 3)] for i in range(ntri + 1)]
    tris = [[0, 1 + i, 2 + i] for i in range(ntri)]
    sch = capi.SCHEME_SBP if scheme == "sbp" else capi.SCHEME_HYBRIDIZED
    c = capi.Case("smooth", scheme=sch, N=4, mesh=dict(verts=verts, tris=tris, domain=(0.0, 0.0, 2.0, 2.0)))
    assert c.K == ntri
    cd = case_dict(c)
    u = c.u0()
    ref, err, _ = Oracle(cd).rhs(u)
    assert err == 0
    h = c.handle(mode=capi.MODE_FAST)
    assert_fast_rhs(h.rhs(u), ref, cd, u)
    dt = 0.5 * c.dt
    u_ref, _, err = Oracle(cd).step_lsrk45(u, np.zeros_like(u), dt, 3)
    assert err == 0
    h.set_state(u)
    h.step(dt, 3)
    assert rel(h.get_state()[0], u_ref) <= RUN_TOL


@pytest.mark.parametrize("name", ["modal_n4_warp", "modal_n3_warp"])
def test_modal_rhs_device_unaligned_input_plain_load_path(name):
    """The modal pair kernels (N=4, N=3) stage a pair's u/gf/b blocks by bulk copies when
    every base pointer is 16 B aligned; a caller's rhs_device input 8 B past a 16 B boundary
    takes the plain-load staging path instead: bitwise the aligned result."""
    import torch

    c = load_golden(name)
    h = make(c, capi.MODE_FAST)
    u = np.ascontiguousarray(c["u"], dtype=np.float64)
    n = u.size
    buf = torch.empty(n + 1, dtype=torch.float64, device="cuda")
    ua, uu = buf[:n], buf[1:]
    out = []
    for view in (ua, uu):
        view.copy_(torch.from_numpy(u.ravel()))
        du = torch.empty(n, dtype=torch.float64, device="cuda")
        h.rhs_device(view.data_ptr(), du.data_ptr())
        torch.cuda.synchronize()
        out.append(du.cpu().numpy().reshape(u.shape))
    assert uu.data_ptr() % 16 == 8
    np.testing.assert_array_equal(out[0], out[1])
    assert_fast_rhs(out[0], c["du_lf"], c, c["u"])


def test_n3_pair_kernel_odd_element_count_within_tolerance():
    """FAST N=3 pair kernel on a curved C4-generator mesh with an even element count per row
    but odd pair-tail handling (K = 162): within the FAST tolerance of the C oracle."""
    c = capi.Case("smooth", N=3, nx=9, warp=0.1)  # K = 162
    cd = case_dict(c)
    u = c.u0()
    ref, err, _ = Oracle(cd).rhs(u)
    assert err == 0
    assert_fast_rhs(c.handle(mode=capi.MODE_FAST).rhs(u), ref, cd, u)
