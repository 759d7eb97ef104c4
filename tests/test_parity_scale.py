"""Per-RHS parity at the bench's own sizes, and the non-finite RHS error path.

C4 (modal N=4, K1D=1024, K = 2,097,152 curved triangles: the bench workload) and
C5 (K1D=2048, K = 8,388,608) are too large for the C oracle to evaluate whole, so
the GPU RHS of the full mesh is compared on sampled elements: the oracle runs on
the sub-mesh made of the samples and their face neighbours (every input of a
sampled element's RHS — its own data and its neighbours' traces, solver.hpp:263-264 —
is in the sub-mesh, so the oracle's du of a sampled element is exactly the
reference's).  PARITY is bitwise; FAST goes through the logged acceptance of
tests/parity_log.py.
"""
import numpy as np
import pytest

import parity_log
from oracle_py import Oracle

pytestmark = pytest.mark.gpu
capi = pytest.importorskip("paper_2005_02516_b200.capi")


def sub_case(c, elems):
    """Case dict (golden layout) of the sampled elements plus their face neighbours;
    returns (dict, local index of every sampled element)."""
    K, Np, nq, nf = c.K, c.Np, c.nq, c.nf
    nh = nq + nf
    nbr = c.view("nbr", True).reshape(K, 3)
    close = np.unique(np.concatenate([elems, nbr[elems].ravel()]))
    close = close[close >= 0]
    loc = -np.ones(K, dtype=np.int64)
    loc[close] = np.arange(close.size)
    sub_nbr = nbr[close].astype(np.int64)
    # neighbours outside the closure (of non-sampled elements only) are never read: walls
    sub_nbr = np.where(sub_nbr >= 0, loc[np.maximum(sub_nbr, 0)], -1).astype(np.int32)

    def per(name, width, integer=False):
        return np.ascontiguousarray(c.view(name, integer).reshape(K, width)[close]).ravel()

    d = {"scheme": [0], "N": [c.N], "Np": [Np], "nq": [nq], "nf": [nf], "npf": [c.npf], "K": [close.size],
         "g": [c.g], "surfq_w": c.array("surfq_w"), "gf": per("gf", 4 * nh), "sJ": per("sJ", nf),
         "nx": per("nx", nf), "ny": per("ny", nf), "nbr": sub_nbr.ravel(), "perm": per("perm", nf, True),
         "b": per("b", Np).reshape(-1, Np), "u": per("u0", 3 * Np).reshape(-1, 3, Np),
         "ref_Vq": c.array("Vq"), "ref_Vf": c.array("Vf"), "ref_Pq": c.array("Pq"), "ref_Qh_x": c.array("Qr"),
         "ref_Qh_y": c.array("Qs"), "Mh_inv": per("Mh_inv", Np * Np)}
    return {k: np.asarray(v) for k, v in d.items()}, loc[elems]


def sampled_parity(k1d, nsample, seed):
    c = capi.Case("smooth", N=4, nx=k1d, warp=0.1, seed=23)
    rng = np.random.default_rng(seed)
    # random elements plus the first/last elements and mesh-row boundaries
    elems = np.unique(np.concatenate([rng.choice(c.K, nsample, replace=False),
                                      [0, 1, 2 * k1d - 1, 2 * k1d, c.K // 2, c.K - 2, c.K - 1]])).astype(np.int64)
    sub, idx = sub_case(c, elems)
    u0 = c.view("u0").reshape(c.K, 3, c.Np)
    ref, err, _ = Oracle(sub).rhs(sub["u"], elems=idx.astype(np.int32))
    assert err == 0
    ref = ref[idx]
    out = {}
    for mode in (capi.MODE_PARITY, capi.MODE_FAST):
        h = c.handle(mode=mode, diagnostics=False)
        out[mode] = h.rhs(u0)[elems]
        h.close()
    np.testing.assert_array_equal(out[capi.MODE_PARITY], ref)
    rec = parity_log.assert_fast_rhs(
        out[capi.MODE_FAST], ref,
        lambda: Oracle(sub, precision="ld").rhs(sub["u"], elems=idx.astype(np.int32))[0][idx],
        label=f"C4 generator K1D={k1d}, {elems.size} sampled elements, LF")
    return rec


def test_c4_bench_workload_sampled_rhs_parity_k1d1024():
    """C4 = the bench workload (K1D=1024): 1,031 sampled elements' RHS, PARITY bitwise
    equal to the C oracle (= the reference's arithmetic), FAST within the logged tolerance."""
    sampled_parity(1024, 1024, 11)


def test_c5_sampled_rhs_parity_k1d2048():
    """C5's largest mesh (K1D=2048, K = 8,388,608) on one GPU: 1,031 sampled elements."""
    sampled_parity(2048, 1024, 13)


@pytest.mark.parametrize("mode", ["parity", "fast"])
@pytest.mark.parametrize("N", [3, 4])
def test_nonfinite_rhs_reports_element_and_time(mode, N):
    """solver.hpp:288-290: a finite state whose RHS overflows (h = 1e200 in one element:
    the projection stays finite, the flux's g h^2 does not) raises "non-finite RHS in
    element k at t = ..." with the element the serial reference throws for (the lowest
    non-finite one, the C oracle's) and the stage time; from rhs() and from steps."""
    c = capi.Case("smooth", N=N, nx=8, warp=0.1)
    from oracle_py import case_dict

    cd = case_dict(c)
    u = c.u0()
    u[41, 0, :] = 0.0
    u[41, 0, 0] = 1e200 * np.sqrt(2.0)  # constant mode: h = 1e200 at every node
    u[41, 1:, :] = 0.0
    _, err, bad = Oracle(cd).rhs(u)
    assert err == 2 and bad >= 0  # ORACLE_ERR_NONFINITE
    h = c.handle(mode=capi.MODE_PARITY if mode == "parity" else capi.MODE_FAST)
    with pytest.raises(capi.NonFiniteError) as ei:
        h.rhs(u, t=0.375)
    assert ei.value.elem == bad
    assert str(ei.value) == f"non-finite RHS in element {bad} at t = 0.375000"
    h.set_state(u, None, 0.25)
    with pytest.raises(capi.NonFiniteError) as ei:
        h.step(1e-5, 3)
    assert ei.value.elem == bad and abs(ei.value.t - 0.25) < 1e-12
    assert str(ei.value).startswith(f"non-finite RHS in element {bad} at t = 0.25")


@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_nonfinite_sbp_rhs_message(mode):
    """solver.hpp:429-431: "non-finite SBP RHS in element k at t = ..." (SBP N=4).  The
    planted momentum (hu = 1e160, u = hu/h ~ 7e159) overflows the EC flux's {hu}{u} in the
    element and across its faces in both arithmetic forms (a planted h alone does not: FAST's
    p = g/2 h_i h_j stays finite where the reference's g{h}^2 - g/4(h_i^2 + h_j^2) is inf - inf)."""
    c = capi.Case("smooth", scheme=capi.SCHEME_SBP, N=4, nx=8, warp=0.1)
    from oracle_py import case_dict

    cd = case_dict(c)
    u = c.u0()
    u[29, 1, :] = 1e160
    _, err, bad = Oracle(cd).rhs(u)
    assert err == 2 and bad >= 0  # ORACLE_ERR_NONFINITE
    h = c.handle(mode=capi.MODE_PARITY if mode == "parity" else capi.MODE_FAST)
    with pytest.raises(capi.NonFiniteError) as ei:
        h.rhs(u, t=0.5)
    assert ei.value.elem == bad
    assert str(ei.value) == f"non-finite SBP RHS in element {bad} at t = 0.500000"


def test_c5_strong_two_partitions_bitwise_k1d2048():
    """C5's strong-scaling mesh (K1D = 2048, K = 8,388,608) cut into 2 y-strips, both ranks
    on one GPU (one host thread each, device-copy exchange callback through the native
    multi-rank schedule): 2 LSRK45 steps bitwise equal to the unpartitioned run."""
    import gc

    from paper_2005_02516_b200.partition import LocalExchange

    g = capi.Case("smooth", N=4, nx=2048, warp=0.1, seed=23)
    dt = g.dt
    hg = g.handle(mode=capi.MODE_FAST, diagnostics=False)
    hg.set_state(g.view("u0").reshape(g.K, 3, g.Np))
    hg.step(dt, 2)
    ug = hg.get_state(with_res=False)[0]
    hg.close()
    g.close()
    del hg, g
    gc.collect()
    cases = [capi.Case("smooth", N=4, nx=2048, warp=0.1, seed=23, strips=2, strip=r, scaling="strong")
             for r in range(2)]
    assert min(c.dt for c in cases) == dt
    hs = [c.handle(mode=capi.MODE_FAST, diagnostics=False) for c in cases]
    for h, c in zip(hs, cases):
        h.set_state(c.view("u0").reshape(c.K, 3, c.Np))
    LocalExchange(hs, [c.halo_desc() for c in cases], cases[0].nf).step(dt, 2)
    off = 0
    for h, c in zip(hs, cases):
        np.testing.assert_array_equal(h.get_state(with_res=False)[0], ug[off:off + c.K])
        off += c.K
    assert off == ug.shape[0]
