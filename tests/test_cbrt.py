"""The friction cube root (kernels.py:240-241).

The oracle's cbrt is correctly rounded (checked against exact rationals) and
the product's host twin is bitwise equal to it; the device cbrt is checked in
test_gpu_parity.py.  On this host numpy's SVML np.cbrt differs in ~0.5 % of
inputs — the reason parity is pinned against the cbrt-aligned reference."""

import math
from fractions import Fraction

import numpy as np
import pytest


def _inputs(n=4000, seed=0):
    rng = np.random.default_rng(seed)
    x = np.exp(rng.uniform(np.log(1e-6), np.log(1e5), n))
    k = np.arange(-40, 40, dtype=float)
    special = np.concatenate([2.0 ** k, np.nextafter(2.0 ** k, 0), np.nextafter(2.0 ** k, np.inf),
                              [1e-5, 8.0, 27.0, 0.125, 1 / 3, 5e-324, 1e-310, 1e300, 1.7e308]])
    return np.concatenate([x, special])


def test_oracle_cbrt_correctly_rounded(oracle_mod):
    x = _inputs()
    y = oracle_mod.cbrt(x)
    for xi, yi in zip(x, y):
        X, Y = Fraction(float(xi)), Fraction(float(yi))
        up = Fraction(math.ulp(float(yi)))
        dn = Fraction(math.ulp(float(np.nextafter(yi, 0))))
        assert (Y - dn / 2) ** 3 <= X <= (Y + up / 2) ** 3, float(xi)


def test_host_twin_bitwise_equals_oracle(oracle_mod):
    from paper_2408_07609_b200 import _native
    x = np.concatenate([_inputs(200000, 1), -_inputs(2000, 2)])
    a, b = _native.cbrt_host(x), oracle_mod.cbrt(x)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_cbrt_special_values(oracle_mod):
    from paper_2408_07609_b200 import _native
    x = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, -8.0, 27.0])
    for y in (oracle_mod.cbrt(x), _native.cbrt_host(x)):
        assert y[0] == 0 and not np.signbit(y[0]) and np.signbit(y[1])
        assert y[2] == np.inf and y[3] == -np.inf and np.isnan(y[4])
        assert y[5] == -2.0 and y[6] == 3.0
