"""Pins of the oracle's phi-solve, Eq. (31)-(33): residual, dense linear solve, closed forms."""
import numpy as np
import pytest


def periodic_apply(phi, tau, mu):
    """(1 - tau mu Delta_per) phi with the 5-point Laplacian of Eq. (35), periodic wrap."""
    lap = (np.roll(phi, 1, 0) + np.roll(phi, -1, 0) + np.roll(phi, 1, 1) + np.roll(phi, -1, 1) - 4 * phi)
    return phi - tau * mu * lap


@pytest.mark.parametrize("taumu", [(0.1, 1.0), (0.1, 8.0), (0.5, 10.0)])
def test_residual_below_1e_10(orc, taumu):
    """North star: the residual of the phi linear system stays below 1e-10."""
    tau, mu = taumu
    rng = np.random.default_rng(int(tau * 100 + mu))
    for trial in range(25):
        F = rng.standard_normal((64, 64))
        phi = orc.solve(F, tau, mu)
        res = np.linalg.norm(periodic_apply(phi, tau, mu) - F) / np.linalg.norm(F)
        assert res < 1e-10


@pytest.mark.parametrize("M,N", [(8, 8), (16, 8), (4, 16)])
def test_dense_solve(orc, M, N):
    """Independent of any FFT: assemble the (MN)^2 periodic system and numpy.linalg.solve it."""
    tau, mu = 0.1, 8.0
    n = M * N
    A = np.zeros((n, n))
    for i in range(M):
        for j in range(N):
            r = i * N + j
            A[r, r] += 1 + 4 * tau * mu
            for di, dj in ((1, 0), (-1, 0), (0, 1), (0, -1)):
                A[r, ((i + di) % M) * N + (j + dj) % N] -= tau * mu
    rng = np.random.default_rng(M + N)
    F = rng.standard_normal((M, N))
    ref = np.linalg.solve(A, F.ravel()).reshape(M, N)
    assert np.max(np.abs(orc.solve(F, tau, mu) - ref)) < 1e-12


def test_constant_and_cos_mode(orc):
    M, N, tau, mu = 32, 16, 0.1, 8.0
    assert np.allclose(orc.solve(np.full((M, N), 0.7), tau, mu), 0.7, atol=1e-14)   # sigma(0,0) = 1
    ii, jj = np.meshgrid(np.arange(M), np.arange(N), indexing="ij")
    for k1, k2 in ((1, 0), (3, 5), (M // 2, N // 2), (0, N // 2)):
        F = np.cos(2 * np.pi * (k1 * ii / M + k2 * jj / N))
        sig = 1 + tau * mu * (4 - 2 * np.cos(2 * np.pi * k1 / M) - 2 * np.cos(2 * np.pi * k2 / N))
        assert np.allclose(orc.solve(F, tau, mu), F / sig, atol=1e-13)
        assert orc.symbol(M, N, tau, mu, k1, k2) == pytest.approx(sig, rel=1e-15)


def test_mean_preserved_and_symbol_range(orc):
    rng = np.random.default_rng(11)
    F = rng.standard_normal((16, 32))
    assert orc.solve(F, 0.1, 8.0).mean() == pytest.approx(F.mean(), abs=1e-14)
    vals = [orc.symbol(16, 32, 0.1, 8.0, a, b) for a in range(16) for b in range(32)]
    assert min(vals) == pytest.approx(1.0) and max(vals) == pytest.approx(1 + 8 * 0.8)
