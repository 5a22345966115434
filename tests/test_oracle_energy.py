"""Pins of the oracle's Eq. (22) energy terms (NEXT-1 monitoring): closed forms on plateaus and on
an impulse, the repulsion double sum by brute force over all pixel pairs, and descent: one phi
sweep with a small time step lowers E1 = gamma E_g + alpha E_a + beta E_r + E_pen at fixed (w, b)
(the sweep is a semi-implicit gradient flow of E1, Eq. 24-26)."""
import math

import numpy as np
import pytest


def _p(window=3, **kw):
    from synth import paper_params
    return paper_params(window, **kw)


def test_plateaus(orc):
    P = _p()
    z = np.zeros((9, 7))
    g = np.random.default_rng(0).uniform(0.1, 1, (9, 7))
    eg, ea, er, ep = orc.energy(P, -np.ones((9, 7)), z, z, z, z, g)   # inside everywhere
    assert (eg, er, ep) == (0.0, 0.0, 0.0) and ea == pytest.approx(g.sum(), rel=1e-14)
    eg, ea, er, ep = orc.energy(P, np.ones((9, 7)), z, z, z, z, g)    # outside everywhere
    assert (eg, ea, er, ep) == (0.0, 0.0, 0.0, 0.0)


def test_impulse(orc):
    """phi = 0 (h = 1, delta = 1/eps, H = 1/2), one w at c, b = 0."""
    P = _p()
    M, N = 11, 12
    z = np.zeros((M, N))
    w1 = z.copy()
    w2 = z.copy()
    w1[5, 6], w2[5, 6] = 0.6, -0.8                 # |w_c| = 1
    g = np.full((M, N), 0.5)
    eg, ea, er, ep = orc.energy(P, z, w1, w2, z, z, g)
    assert eg == pytest.approx(0.5 * 1.0 / P["epsilon"])
    assert ea == pytest.approx(0.5 * 0.5 * M * N)
    assert er == pytest.approx(-1.0)               # -G(0) |w_c|^2 h(0)^2
    assert ep == pytest.approx(P["mu"] / 2 * 1.0)


def test_repulsion_double_sum_brute_force(orc):
    rng = np.random.default_rng(3)
    P = _p(window_shape=1, window=20, d=2.0)       # window covers the grid: all pairs
    M, N = 6, 5
    phi = rng.uniform(-1, 1, (M, N))
    w1, w2 = rng.uniform(-1, 1, (M, N)), rng.uniform(-1, 1, (M, N))
    z = np.zeros((M, N))
    _, _, er, _ = orc.energy(P, phi, w1, w2, z, z, np.ones((M, N)))
    hv = np.vectorize(lambda x: orc.h(x, P["epsilon"], P["l"]))(phi)
    ref = 0.0
    for i in range(M):
        for j in range(N):
            for k in range(M):
                for l in range(N):
                    G = math.exp(-((i - k) ** 2 + (j - l) ** 2) / P["d"] ** 2)
                    ref -= G * (w1[i, j] * w1[k, l] + w2[i, j] * w2[k, l]) * hv[i, j] * hv[k, l]
    assert er == pytest.approx(ref, rel=1e-12)


def test_sweep_descends_E1(orc):
    rng = np.random.default_rng(5)
    P = _p(tau=1e-3)
    M = N = 16
    ii, jj = np.meshgrid(np.arange(M), np.arange(N), indexing="ij")
    phi = 0.9 * np.tanh((np.hypot(ii - 7.5, jj - 7.5) - 4.0) / 2.0)
    w1, w2 = orc.grad(phi)
    w1 = w1 + 0.05 * rng.standard_normal((M, N))
    w2 = w2 + 0.05 * rng.standard_normal((M, N))
    b1, b2 = 0.05 * rng.standard_normal((M, N)), 0.05 * rng.standard_normal((M, N))
    g = rng.uniform(0.2, 1, (M, N))

    def E1(ph):
        eg, ea, er, ep = orc.energy(P, ph, w1, w2, b1, b2, g)
        return P["gamma"] * eg + P["alpha"] * ea + P["beta"] * er + ep
    new = orc.sweep(P, phi, w1, w2, b1, b2, g)
    assert E1(new) < E1(phi)
