"""The exact accumulator behind the device diagnostics (csrc/exact_sum.h), host
side: its correctly rounded sum equals Python's math.fsum bit for bit on
adversarial inputs (cancellation, ties, huge/tiny/subnormal terms), and the
raw-record merge is exact.  CPU only (no compute call touches the GPU)."""
import math

import numpy as np
import pytest

from paper_2005_02516_b200 import capi


def cases():
    rng = np.random.default_rng(0)
    for trial in range(240):
        n = int(rng.integers(1, 3000))
        kind = trial % 6
        if kind == 0:
            x = rng.standard_normal(n)
        elif kind == 1:
            x = rng.standard_normal(n) * 10.0 ** rng.integers(-300, 300, n)
        elif kind == 2:  # near-total cancellation
            x = rng.standard_normal(n)
            x = np.r_[x, -x[::-1]][:n]
            x[0] += 1e-30
        elif kind == 3:  # tiny and subnormal
            x = rng.standard_normal(n) * 2.0 ** -1000
        elif kind == 4:  # near overflow
            x = np.r_[1e308, 5e307, -1e308, rng.standard_normal(n)]
        else:  # rounding ties and sticky bits
            x = np.r_[1.0, 2.0 ** -53, 2.0 ** -53 * (1 + 2.0 ** -52), -1.0, rng.standard_normal(n) * 2.0 ** -60]
        yield x
    for x in ([1.0, 2.0 ** -53], [1.0, 2.0 ** -53, 2.0 ** -200], [1.0 + 2.0 ** -52, 2.0 ** -53],
              [-1.0, -(2.0 ** -53)], [5e-324] * 5, [1e-310, -3e-310], [0.0, -0.0], []):
        yield np.array(x, dtype=np.float64)


def test_exact_sum_equals_fsum():
    for x in cases():
        assert capi.exact_sum(x) == math.fsum(x.tolist()), x[:4]


def test_exact_sum_order_independent():
    rng = np.random.default_rng(5)
    x = rng.standard_normal(20000) * 10.0 ** rng.integers(-20, 20, 20000)
    s = capi.exact_sum(x)
    for _ in range(5):
        assert capi.exact_sum(rng.permutation(x)) == s


def test_exact_sum_rejects_nonfinite():
    with pytest.raises(capi.SwedgError):
        capi.exact_sum(np.array([1.0, np.inf]))
