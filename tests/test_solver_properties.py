"""The reference's hot-path property tests (proj/tests/test_solver.cpp) on the GPU path,
for the production FAST kernels of every degree and for PARITY: entropy projection of a
constant state (:96-110), projection convergence rate (:112-135) and mass conservation
with walls (:238-246).  Free stream, lake at rest, entropy balance and positivity are in
test_configs.py / test_gpu_parity.py."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
capi = pytest.importorskip("paper_2005_02516_b200.capi")

MODES = [("fast", capi.MODE_FAST), ("parity", capi.MODE_PARITY)]


def uniform_mesh(n, lo=-1.0, hi=1.0):
    """uniform_tri_mesh(n, n, [lo,hi]^2) vertex and triangle lists (mesh.hpp:83-108)."""
    verts = [[lo + (hi - lo) * i / n, lo + (hi - lo) * j / n] for j in range(n + 1) for i in range(n + 1)]
    vid = lambda i, j: j * (n + 1) + i  # noqa: E731
    tris = []
    for j in range(n):
        for i in range(n):
            tris += [[vid(i, j), vid(i + 1, j), vid(i + 1, j + 1)], [vid(i, j), vid(i + 1, j + 1), vid(i, j + 1)]]
    return verts, tris


@pytest.mark.parametrize("mode_name,mode", MODES)
@pytest.mark.parametrize("N", [1, 2, 3, 4])
def test_entropy_projection_of_a_constant_state_is_exact(N, mode_name, mode):
    """test_solver.cpp:96-110: h = 2, hu = 0.6, hv = 0 (constant modal coefficient) over a
    flat bottom projects to the same state at every stacked point, to 1e-12."""
    c = capi.Case("smooth", N=N, nx=2, warp=0.1)
    h = c.handle(mode=mode, set_bathymetry=False, diagnostics=False)
    h.set_bathymetry(np.zeros((c.K, c.Np)))
    u = np.zeros((c.K, 3, c.Np))
    u[:, 0, 0] = np.sqrt(2.0) * 2.0
    u[:, 1, 0] = np.sqrt(2.0) * 0.6
    p = h.entropy_projection(u)
    np.testing.assert_allclose(p[:, 0], 2.0, rtol=1e-12)
    np.testing.assert_allclose(p[:, 1], 0.6, rtol=1e-12)
    assert np.abs(p[:, 2]).max() < 1e-12


@pytest.mark.parametrize("mode_name,mode", MODES)
@pytest.mark.parametrize("N", [2, 3, 4])
def test_entropy_projection_converges_at_the_projection_rate(N, mode_name, mode):
    """test_solver.cpp:112-135: max |proj - [Vq; Vf] u| on 4x4 and 8x8 affine meshes
    (smooth_state seed 5, flat bottom) decreases at a rate > N + 0.5."""
    errs = []
    for n in (4, 8):
        c = capi.Case("smooth", N=N, nx=n, warp=0.0, seed=5)
        h = c.handle(mode=mode, set_bathymetry=False, diagnostics=False)
        h.set_bathymetry(np.zeros((c.K, c.Np)))
        u = c.u0()
        p = h.entropy_projection(u)
        Vq = c.array("Vq").reshape(c.Np, c.nq).T
        Vf = c.array("Vf").reshape(c.Np, c.nf).T
        direct = np.concatenate([np.einsum("qm,kcm->kcq", Vq, u), np.einsum("qm,kcm->kcq", Vf, u)], axis=2)
        errs.append(np.abs(p - direct).max())
    assert np.log2(errs[0] / errs[1]) > N + 0.5, errs


@pytest.mark.parametrize("mode_name,mode", MODES)
@pytest.mark.parametrize("N", [2, 3, 4])
def test_walls_conserve_mass(N, mode_name, mode):
    """test_solver.cpp:238-246: a 4x4 mesh whose boundary faces are all walls (connect with
    no periodicity), flat bottom, smooth state seed 31: the RHS conserves mass to 1e-10."""
    verts, tris = uniform_mesh(4)
    c = capi.Case("smooth", N=N, seed=31, mesh=dict(verts=verts, tris=tris, domain=(0.0, 0.0, 2.0, 2.0)))
    assert (c.iarray("nbr") < 0).sum() == 16  # 4 faces x 4 sides
    h = c.handle(mode=mode, set_bathymetry=False, diagnostics=False)
    h.set_bathymetry(np.zeros((c.K, c.Np)))
    du = h.rhs(c.u0())
    w = c.array("volq_w")
    J = c.array("J_vol").reshape(c.K, c.nq)
    Vq = c.array("Vq").reshape(c.Np, c.nq).T
    rate = float((w[None, :] * J * (du[:, 0, :] @ Vq.T)).sum())
    assert abs(rate) < 1e-10, rate
