"""R_GPU study kernels (bench.hpp:55-128) on the GPU: PARITY bit-for-bit equal to the
reference's kernel_matvec / kernel_fluxdiff / kernel_fluxdiff_skew outputs (golden
fixture from the unmodified reference, n = 6..50), FAST within 1e-12 relative;
larger n against the C oracle."""
import numpy as np
import pytest

from oracle_py import load_golden, ratio_kernels

pytestmark = pytest.mark.gpu
capi = pytest.importorskip("paper_2005_02516_b200.capi")


def rel(a, b):
    return np.abs(a - b).max() / (1.0 + np.abs(b).max())


@pytest.mark.parametrize("mode", ["parity", "fast"])
def test_ratio_kernels_vs_reference_fixture(mode):
    G = load_golden("ratio")
    m = capi.MODE_PARITY if mode == "parity" else capi.MODE_FAST
    for n in G["sizes"]:
        p = f"n{n}_"
        _, _, ydg, yes = capi.ratio_kernels(G[p + "Q"], G[p + "u"], mode=m, reps=1)
        nq = int(G[p + "nq"][0])
        Qz = np.array(G[p + "Q"], copy=True)
        Qz[nq:, nq:] = 0.0
        _, _, _, ysk = capi.ratio_kernels(Qz, G[p + "u"], nq=nq, mode=m, reps=1)
        if mode == "parity":
            np.testing.assert_array_equal(ydg, G[p + "y_dg"])
            np.testing.assert_array_equal(yes, G[p + "y_esdg"])
            np.testing.assert_array_equal(ysk, G[p + "y_skew"])
        else:
            assert rel(ydg, G[p + "y_dg"]) <= 1e-12
            assert rel(yes, G[p + "y_esdg"]) <= 1e-12
            assert rel(ysk, G[p + "y_skew"]) <= 1e-12


@pytest.mark.parametrize("n", [100, 200])
def test_ratio_kernels_large_n_vs_oracle(n):
    rng = np.random.default_rng(n)
    K = 37
    Q = rng.uniform(-1, 1, (n, n))
    h = rng.uniform(0.5, 2.0, (K, n))
    u = np.stack([h, h * rng.uniform(-1, 1, (K, n)), h * rng.uniform(-1, 1, (K, n))], axis=1)
    dg, es = ratio_kernels(Q, u)
    _, _, ydg, yes = capi.ratio_kernels(Q, u, mode=capi.MODE_PARITY, reps=1)
    np.testing.assert_array_equal(ydg, dg)
    np.testing.assert_array_equal(yes, es)
    _, _, ydg, yes = capi.ratio_kernels(Q, u, mode=capi.MODE_FAST, reps=1)
    assert rel(ydg, dg) <= 1e-12 and rel(yes, es) <= 1e-12
