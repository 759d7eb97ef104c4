"""BASELINE.json configs on the GPU, built by the native setup.

C1 (vortex N=3 K1D=16) and the small C2/C3 cases are pinned bitwise by
test_gpu_parity.py (golden fixtures).  Here: the configs at their stated sizes
(C2 K=512 curved lake to t=0.5, C3 SBP N=4 dam break K1D=128, C4 K1D=1024) —
parity against the C oracle where the oracle finishes in seconds, and
size-independent properties (well-balancedness, free stream, mass
conservation, positivity) at full size.
"""
import numpy as np
import pytest

import parity_log
from oracle_py import Oracle, case_dict

pytestmark = pytest.mark.gpu
capi = pytest.importorskip("paper_2005_02516_b200.capi")


def mass_rate(case, du):
    """sum_k int du_h (conservation_rate, solver.hpp:543-563)."""
    w = case.array("volq_w")
    J = case.array("J_vol").reshape(case.K, case.nq)
    if case.scheme == capi.SCHEME_SBP:
        return float((w[None, :] * J * du[:, 0, :]).sum())
    Vq = case.array("Vq").reshape(case.Np, case.nq).T
    return float((w[None, :] * J * (du[:, 0, :] @ Vq.T)).sum())


def test_c2_lake_at_rest_k512_to_t05():
    """C2: N=3 curved (warp 0.1) lake at rest, 16x16 (K=512), to t=0.5: deviation <= 1e-9
    (acceptance.cpp:96-117 bound), both arithmetic modes."""
    c = capi.Case("lake", N=3, nx=16, warp=0.1)
    u0 = c.u0()
    nsteps = int(np.ceil(0.5 / c.dt - 1e-12))
    for mode in (capi.MODE_PARITY, capi.MODE_FAST):
        h = c.handle(mode=mode)
        h.set_state(u0)
        t = 0.0
        for _ in range(nsteps):
            dt = min(c.dt, 0.5 - t)
            h.step(dt, 1, sync=False)
            t += dt
        h.check()
        u, _, _ = h.get_state()
        assert np.abs(u - u0).max() < 1e-9


def test_c3_sbp_dambreak_k1d128():
    """C3: SBP N=4 dam break, 128x128 (K=32,768): PARITY rhs bit-for-bit equal to the C
    oracle; FAST within the accuracy criterion; 100 steps stay positive and conserve mass."""
    c = capi.Case("dambreak", scheme=capi.SCHEME_SBP, N=4, nx=128, cfl=0.0625)
    assert c.K == 32768 and c.nq == 37
    cd = case_dict(c)
    u0 = c.u0()
    ref, err, _ = Oracle(cd).rhs(u0)
    assert err == 0
    hp = c.handle(mode=capi.MODE_PARITY)
    np.testing.assert_array_equal(hp.rhs(u0), ref)
    hf = c.handle(mode=capi.MODE_FAST)
    du = hf.rhs(u0)
    parity_log.assert_fast_rhs(du, ref, lambda: Oracle(cd, precision="ld").rhs(u0)[0], label="C3 K1D=128 LF")
    assert abs(mass_rate(c, du)) < 1e-9
    hf.set_state(u0)
    hf.step(c.dt, 100)
    u, _, _ = hf.get_state()
    assert np.isfinite(u).all() and u[:, 0, :].min() > 0.0
    w = c.array("volq_w")
    J = c.array("J_vol").reshape(c.K, c.nq)
    m0 = (w * J * u0[:, 0, :]).sum()
    m1 = (w * J * u[:, 0, :]).sum()
    assert abs(m1 - m0) / m0 < 1e-12


def test_c4_sample_parity_k1d256():
    """C4 workload generator (smooth wave + lake bathymetry, curved, N=4) at K1D=256:
    PARITY rhs of 512 sampled elements bit-for-bit equal to the C oracle; FAST within
    1e-12 relative or — the reference's own rounding error grows like 1/h (SURVEY §0:
    ~1e-12 at K1D=128) — no less accurate than the reference against long double."""
    c = capi.Case("smooth", N=4, nx=256, warp=0.1)
    cd = case_dict(c)
    u0 = c.u0()
    h = c.handle(mode=capi.MODE_FAST)
    du = h.rhs(u0)
    rng = np.random.default_rng(3)
    elems = np.sort(rng.choice(c.K, 512, replace=False)).astype(np.int32)
    ref, err, _ = Oracle(cd).rhs(u0, elems=elems)
    assert err == 0
    parity_log.assert_fast_rhs(du[elems], ref[elems],
                               lambda: Oracle(cd, precision="ld").rhs(u0, elems=elems)[0][elems],
                               label="C4 generator K1D=256, 512 sampled elements, LF")
    hp = c.handle(mode=capi.MODE_PARITY)
    np.testing.assert_array_equal(hp.rhs(u0)[elems], ref[elems])


def test_c4_full_size_properties_k1d1024():
    """C4 at full size (K=2,097,152): lake at rest stays at rest (well-balanced), a
    constant state has zero RHS (free stream), and the smooth-wave RHS conserves mass."""
    lake = capi.Case("lake", N=4, nx=1024, warp=0.1)
    h = lake.handle(mode=capi.MODE_FAST)
    du = h.rhs(lake.u0())
    assert np.abs(du).max() < 1e-9
    h.close()
    sm = capi.Case("smooth", N=4, nx=1024, warp=0.1)
    h = sm.handle(mode=capi.MODE_FAST)
    u = sm.u0()
    du = h.rhs(u)
    assert np.isfinite(du).all()
    scale = np.abs(du).max()
    assert abs(mass_rate(sm, du)) < 1e-10 * max(1.0, scale)
    # free stream: h = 1.7 everywhere, no flow, flat bottom.  The exact RHS is 0; the
    # rounding noise grows like 1/h, so FAST is bounded by the reference's own noise on a
    # sample of elements (C oracle, double).
    free = np.zeros_like(u)
    free[:, 0, 0] = np.sqrt(2.0) * 1.7
    zb = np.zeros((sm.K, sm.Np))
    h.set_bathymetry(zb)
    du_free = h.rhs(free)
    cd = case_dict(sm)
    cd["b"] = zb
    elems = np.arange(0, sm.K, sm.K // 256, dtype=np.int32)
    ref, err, _ = Oracle(cd).rhs(free, elems=elems)
    assert err == 0
    noise_ref = np.abs(ref[elems]).max()
    assert noise_ref < 1e-8
    assert np.abs(du_free).max() <= 8.0 * noise_ref


def _entropy_vars(h, hu, hv, b, g):
    vx, vy = hu / h, hv / h
    return g * (h + b) - 0.5 * (vx * vx + vy * vy), vx, vy


@pytest.mark.parametrize("N", [3, 4])
def test_fast_modal_entropy_balance_and_mass_k1d64(N):
    """The reference's semi-discrete entropy balance (test_solver.cpp:172-206) for the
    FAST N=3 and N=4 pair kernels on a curved K1D=64 mesh: entropy-conservative flux ->
    sum_k v_h^T M_h du ~ 0 (1e-9 of the RHS scale), Lax-Friedrichs -> <= 0,
    mass conserved by both (entropy_rate / conservation_rate, solver.hpp:503-563)."""
    c = capi.Case("smooth", N=N, nx=64, warp=0.1)
    K, Np, nq = c.K, c.Np, c.nq
    u = c.u0()
    Vq = c.array("Vq").reshape(Np, nq).T
    Pq = c.array("Pq").reshape(nq, Np).T
    w = c.array("volq_w")
    J = c.array("J_vol").reshape(K, nq)
    uq = np.einsum("qm,kcm->kcq", Vq, u)
    bq = c.b() @ Vq.T
    v1, v2, v3 = _entropy_vars(uq[:, 0], uq[:, 1], uq[:, 2], bq, c.g)
    vh = np.stack([v1 @ Pq.T, v2 @ Pq.T, v3 @ Pq.T], axis=1)           # [K][3][Np]
    rates = {}
    for pen in (capi.PENALTY_EC, capi.PENALTY_LF):
        h = c.handle(mode=capi.MODE_FAST, penalty=pen)
        du = h.rhs(u)
        duq = np.einsum("qm,kcm->kcq", Vq, du)                          # M_h du = Vq^T wJ Vq du
        mdu = np.einsum("qm,kcq->kcm", Vq, (w[None, :] * J)[:, None, :] * duq)
        rates[pen] = (float((vh * mdu).sum()), float(np.abs(du).max()))
        assert abs(float(((w[None, :] * J) * duq[:, 0]).sum())) < 1e-10 * (1 + rates[pen][1])
        h.close()
    r_ec, scale = rates[capi.PENALTY_EC]
    assert abs(r_ec) < 1e-9 * (1.0 + scale)
    assert rates[capi.PENALTY_LF][0] <= 1e-12 * (1.0 + scale)


def test_fast_sbp_entropy_balance_k1d32():
    """test_solver.cpp:208-236 for the FAST SBP N=4 kernel: perturbed lake at rest on a
    curved K1D=32 mesh, sum_k v^T M du ~ 0 with the EC flux, <= 0 with LF, mass kept."""
    c = capi.Case("lake", scheme=capi.SCHEME_SBP, N=4, nx=32, warp=0.1)
    K, nq = c.K, c.nq
    rng = np.random.default_rng(3)
    u = c.u0() + rng.uniform(-0.05, 0.05, (K, 3, nq))
    b = c.b()
    m = c.array("M_diag")[None, :] * c.array("J_vol").reshape(K, nq)
    v = np.stack(_entropy_vars(u[:, 0], u[:, 1], u[:, 2], b, c.g), axis=1)
    rates = {}
    for pen in (capi.PENALTY_EC, capi.PENALTY_LF):
        h = c.handle(mode=capi.MODE_FAST, penalty=pen)
        du = h.rhs(u)
        rates[pen] = (float((m[:, None, :] * v * du).sum()), float(np.abs(du).max()))
        assert abs(float((m * du[:, 0]).sum())) < 1e-10 * (1 + rates[pen][1])
        h.close()
    r_ec, scale = rates[capi.PENALTY_EC]
    assert abs(r_ec) < 1e-9 * (1.0 + scale)
    assert rates[capi.PENALTY_LF][0] <= 1e-12 * (1.0 + scale)


@pytest.mark.parametrize("mode", [capi.MODE_FAST, capi.MODE_PARITY])
def test_acceptance_2_lake_at_rest_all_degrees(mode):
    """Acceptance criterion 2 (acceptance.cpp:96-117) through the device run loop:
    lake at rest, N = 1..4, 8x8 and 16x16, affine and curved, to t = 0.5: L2
    deviation from the discrete steady state <= 1e-9 (the reference's worst: 4.2e-13)."""
    from paper_2005_02516_b200 import run as srun

    worst = 0.0
    for N in range(1, 5):
        for n in (8, 16):
            for warp in (0.0, 0.1):
                c = capi.Case("lake", N=N, nx=n, warp=warp)
                res = srun.run(c, tfinal=0.5, mode=mode)
                worst = max(worst, res["error"]["combined"])
                c.close()
    assert worst <= 1e-9, worst


def test_acceptance_7_dam_break_robustness():
    """Acceptance criterion 7 (acceptance.cpp:279-305): hybridized N = 3 dam break on
    20x20 to t = 1.5 with CFL 0.0625 stays positive (min_h over the invariant series)
    and conserves mass to 1e-8 (reference: min_h 1.146, drift 2.8e-14)."""
    from paper_2005_02516_b200 import run as srun

    c = capi.Case("dambreak", N=3, nx=20, cfl=0.0625)
    res = srun.run(c, tfinal=1.5)
    s = res["series"]
    assert abs(res["t"] - 1.5) < 1e-12
    min_h = s[:, 5].min()
    drift = abs(s[-1, 1] - s[0, 1]) / s[0, 1]
    assert min_h > 0.0 and drift <= 1e-8, (min_h, drift)
    assert abs(min_h - 1.146) < 5e-3, min_h  # the reference's value (3 digits printed)


@pytest.mark.gpu
def test_c3_positivity_loss_matches_reference_arithmetic():
    """C3 toward its horizon: the reference scheme itself (PARITY = the reference's
    arithmetic bit for bit) loses positivity in this dam break at t ~ 0.070 (no limiter in
    the paper's scheme); FAST stops at the same element and stage time with the
    reference's message, after a trajectory equal to PARITY's to rounding."""
    c = capi.Case("dambreak", scheme=capi.SCHEME_SBP, N=4, nx=128, cfl=0.0625)
    stops = []
    for mode in (capi.MODE_PARITY, capi.MODE_FAST):
        h = c.handle(mode=mode)
        h.set_state(c.u0())
        h.step(c.dt, 150)
        u150, _, _ = h.get_state()
        with pytest.raises(capi.PositivityError) as ei:
            h.step(c.dt, 100)
        assert "nonpositive water height in element" in str(ei.value)
        stops.append((ei.value.elem, ei.value.t, u150))
    assert stops[0][0] == stops[1][0]
    assert abs(stops[0][1] - stops[1][1]) < 1e-12
    assert 0.06 < stops[0][1] < 0.08
    u_p, u_f = stops[0][2], stops[1][2]
    assert np.abs(u_f - u_p).max() / (1 + np.abs(u_p).max()) < 1e-10


@pytest.mark.gpu
def test_c4_bench_horizon_fast_vs_reference_arithmetic():
    """The bench workload itself (C4, K = 2,097,152, 25 LSRK45 steps = the bench's warm-up
    plus timed steps): the production FAST path stays within the run tolerance
    (1e-10 relative) of PARITY, the reference's arithmetic bit for bit."""
    c = capi.Case("smooth", N=4, nx=1024, warp=0.1, seed=23)
    outs = []
    for mode in (capi.MODE_PARITY, capi.MODE_FAST):
        h = c.handle(mode=mode)
        h.set_state(c.u0())
        h.step(c.dt, 25)
        outs.append(h.get_state()[0])
        h.close()
    d = np.abs(outs[1] - outs[0]).max() / (1 + np.abs(outs[0]).max())
    assert d <= 1e-10, d
