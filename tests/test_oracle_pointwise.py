"""Pins of the oracle's regularizers (Eq. 5, 6, 11, 28, 29) and edge indicator (Eq. 1).

Pins: closed-form values from tests/golden/regularizers.json, central finite
differences (delta = dH, delta' = d delta, h' = dh), support / range
invariants, and scipy.ndimage's Gaussian filter for the blur in g.
"""
import json
import math
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "regularizers.json")))


@pytest.mark.parametrize("name", ["H", "delta", "delta_prime", "h", "h_prime"])
def test_golden_values(orc, name):
    fn = getattr(orc, name)
    for case in GOLD[name]:
        args = [case["phi"], case["eps"]] + ([case["l"]] if "l" in case else [])
        assert fn(*args) == pytest.approx(case["value"], abs=1e-12), case["cite"]


@pytest.mark.parametrize("eps,l", [(1.0, 1.0), (0.5, 0.5), (0.7, 0.3)])
def test_derivatives_by_finite_differences(orc, eps, l):
    rng = np.random.default_rng(0)
    hstep = 1e-6
    for x in rng.uniform(-(l + eps) * 1.2, (l + eps) * 1.2, 100):
        dH = (orc.H(x + hstep, eps) - orc.H(x - hstep, eps)) / (2 * hstep)
        assert orc.delta(x, eps) == pytest.approx(dH, abs=1e-6)
        dd = (orc.delta(x + hstep, eps) - orc.delta(x - hstep, eps)) / (2 * hstep)
        assert orc.delta_prime(x, eps) == pytest.approx(dd, abs=1e-5 / eps ** 2)
        dh = (orc.h(x + hstep, eps, l) - orc.h(x - hstep, eps, l)) / (2 * hstep)
        assert orc.h_prime(x, eps, l) == pytest.approx(dh, abs=1e-5 / eps)


def test_ranges_and_support(orc):
    eps, l = 0.5, 0.5
    for x in np.linspace(-3, 3, 601):
        assert -1e-15 <= orc.H(x, eps) <= 1.0 + 1e-15  # sin(+-pi) rounds to ~1e-16
        assert orc.delta(x, eps) >= 0.0
        assert -1e-15 <= orc.h(x, eps, l) <= 1.0 + 1e-15
        assert orc.h(x, eps, l) == pytest.approx(orc.h(-x, eps, l), abs=1e-15)  # even
        assert orc.h_prime(x, eps, l) == pytest.approx(-orc.h_prime(-x, eps, l), abs=1e-15)   # odd
        assert orc.delta_prime(x, eps) == pytest.approx(-orc.delta_prime(-x, eps), abs=1e-15)
        if abs(x) > eps:
            assert orc.delta(x, eps) == 0.0 and orc.delta_prime(x, eps) == 0.0
        if abs(x) >= l + eps:
            assert abs(orc.h(x, eps, l)) <= 1e-15 and abs(orc.h_prime(x, eps, l)) <= 1e-15


def test_delta_integrates_to_one(orc):
    """trapezoid integral of delta over [-eps, eps] is 1."""
    for eps in (1.0, 0.5):
        xs = np.linspace(-eps, eps, 20001)
        vals = np.array([orc.delta(x, eps) for x in xs])
        assert np.trapezoid(vals, xs) == pytest.approx(1.0, abs=1e-6)


def test_edge_constant_image(orc):
    g = orc.edge(np.full((16, 12), 0.37), 1.0, 30.0, 2)
    assert np.all(g == 1.0)


def test_edge_linear_ramp_closed_form(orc):
    """Interior of f = a*j: blur keeps the ramp, central difference gives a, so g = 1/(1+rho a^2)."""
    a, rho = 0.2, 25.0                       # rho a^2 = 1 -> g = 0.5
    f = a * np.tile(np.arange(32, dtype=float), (20, 1))
    g = orc.edge(f, 1.0, rho, 2)
    assert np.allclose(g[:, 4:-4], 0.5, atol=1e-12)
    g1 = orc.edge(f, 1.0, rho, 1)            # s = 1: 1/(1 + rho |a|)
    assert np.allclose(g1[:, 4:-4], 1.0 / (1.0 + rho * a), atol=1e-12)


def test_edge_matches_scipy_blur(orc):
    """G_sigma * f with radius ceil(3 sigma), normalized, replicate padding == scipy.ndimage.gaussian_filter."""
    from scipy.ndimage import gaussian_filter
    rng = np.random.default_rng(3)
    f = rng.uniform(0, 1, (24, 40))
    fs = gaussian_filter(f, 1.0, mode="nearest", truncate=3.0)
    gx = np.empty_like(fs)
    gy = np.empty_like(fs)
    gx[1:-1] = (fs[2:] - fs[:-2]) / 2
    gx[0] = (fs[1] - fs[0]) / 2
    gx[-1] = (fs[-1] - fs[-2]) / 2
    gy[:, 1:-1] = (fs[:, 2:] - fs[:, :-2]) / 2
    gy[:, 0] = (fs[:, 1] - fs[:, 0]) / 2
    gy[:, -1] = (fs[:, -1] - fs[:, -2]) / 2
    for rho, s in ((30.0, 2), (5.0, 1)):
        mag = gx ** 2 + gy ** 2
        if s == 1:
            mag = np.sqrt(mag)
        assert np.allclose(orc.edge(f, 1.0, rho, s), 1.0 / (1.0 + rho * mag), atol=1e-13)


def test_edge_step_minimum_on_step(orc):
    """vertical step -> g minimal on the step columns, increasing away from it."""
    f = np.zeros((16, 16))
    f[:, 8:] = 1.0
    g = orc.edge(f, 1.0, 30.0, 2)
    row = g[8]
    assert row.argmin() in (7, 8)
    assert np.all(np.diff(row[:8]) <= 1e-15) and np.all(np.diff(row[8:]) >= -1e-15)
    assert math.isclose(g.min(), g[:, 7].min(), rel_tol=1e-12) or math.isclose(g.min(), g[:, 8].min(), rel_tol=1e-12)
