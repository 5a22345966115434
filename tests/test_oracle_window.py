"""Pins of the oracle's non-local window sum (Eq. 38; readings Q2, Q5)."""
import numpy as np
import pytest


def disc(R):
    return [(p, q) for p in range(-R, R + 1) for q in range(-R, R + 1) if p * p + q * q <= R * R]


def test_disc_tap_counts():
    assert [len(disc(R)) for R in (3, 4, 5, 6)] == [29, 49, 81, 113]


@pytest.mark.parametrize("R", [3, 4, 6])
def test_impulse_response(orc, R):
    """A single w at c with phi = 0 gives v(x) = G(x - c) w_c h(0): the disc of weights."""
    M = N = 2 * R + 9
    u1 = np.zeros((M, N))
    u2 = np.zeros((M, N))
    c = (M // 2, N // 2)
    u1[c], u2[c] = 1.0, -2.0
    v1, v2 = orc.window_sum(u1, u2, R, float(R), 0)
    for i in range(M):
        for j in range(N):
            p, q = i - c[0], j - c[1]
            G = np.exp(-(p * p + q * q) / R ** 2) if p * p + q * q <= R * R else 0.0
            assert v1[i, j] == pytest.approx(G, abs=1e-15)
            assert v2[i, j] == pytest.approx(-2 * G, abs=1e-15)


def test_full_window_equals_double_sum(orc):
    """Square window covering the whole grid == sum_y G(x-y) u(y) over all y."""
    rng = np.random.default_rng(5)
    M, N, d = 6, 5, 2.5
    u1, u2 = rng.standard_normal((M, N)), rng.standard_normal((M, N))
    v1, v2 = orc.window_sum(u1, u2, 12, d, 1)
    ii, jj = np.meshgrid(np.arange(M), np.arange(N), indexing="ij")
    for i in range(M):
        for j in range(N):
            G = np.exp(-((ii - i) ** 2 + (jj - j) ** 2) / d ** 2)
            assert v1[i, j] == pytest.approx(np.sum(G * u1), abs=1e-13)
            assert v2[i, j] == pytest.approx(np.sum(G * u2), abs=1e-13)


def test_locality_and_zero_padding(orc):
    """Perturbing u at y changes v only within the disc around y; out-of-image taps are 0."""
    rng = np.random.default_rng(6)
    M, N, R = 20, 17, 4
    u1, u2 = rng.standard_normal((M, N)), rng.standard_normal((M, N))
    a1, a2 = orc.window_sum(u1, u2, R, float(R), 0)
    u1b = u1.copy()
    u1b[3, 15] += 1.0
    b1, b2 = orc.window_sum(u1b, u2, R, float(R), 0)
    diff = np.argwhere(np.abs(b1 - a1) > 0)
    assert all((i - 3) ** 2 + (j - 15) ** 2 <= R * R for i, j in diff)
    assert np.array_equal(a2, b2)
    # corner pixel: only in-image taps contribute
    s = sum(np.exp(-(p * p + q * q) / R ** 2) * u1[p, q] for p, q in disc(R) if p >= 0 and q >= 0)
    assert a1[0, 0] == pytest.approx(s, abs=1e-13)


def test_reflection_symmetry(orc):
    rng = np.random.default_rng(8)
    u1, u2 = rng.standard_normal((12, 12)), rng.standard_normal((12, 12))
    v1, _ = orc.window_sum(u1, u2, 3, 3.0, 0)
    w1, _ = orc.window_sum(u1[::-1, ::-1].copy(), u2, 3, 3.0, 0)
    assert np.allclose(v1, w1[::-1, ::-1], atol=1e-14)
    t1, _ = orc.window_sum(u1.T.copy(), u2, 3, 3.0, 0)
    assert np.allclose(v1, t1.T, atol=1e-14)
