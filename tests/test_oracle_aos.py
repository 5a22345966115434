"""Pins of the oracle's AOS phi solve (NEXT-4): each 1-D solve against a dense
numpy.linalg.solve of the Neumann tridiagonal system, constants preserved, and consistency of the
AOS splitting with the exact Neumann solve of (1 - tau mu Delta_N) phi = F to O((tau mu)^2)."""
import numpy as np
import pytest


def neumann_A(n):
    A = np.zeros((n, n))
    for i in range(n):
        if i > 0:
            A[i, i - 1] += 1
            A[i, i] -= 1
        if i < n - 1:
            A[i, i + 1] += 1
            A[i, i] -= 1
    return A


@pytest.mark.parametrize("n,c", [(1, 0.8), (2, 0.8), (7, 0.3), (64, 0.8), (33, 5.0)])
def test_thomas_vs_dense(orc, n, c):
    rng = np.random.default_rng(n)
    f = rng.standard_normal(n)
    ref = np.linalg.solve(np.eye(n) - c * neumann_A(n), f)
    assert np.max(np.abs(orc.thomas_neumann(f, c) - ref)) < 1e-13


def test_aos_constant_and_dense(orc):
    tau, mu = 0.05, 8.0
    assert np.allclose(orc.solve_aos(np.full((16, 8), 0.7), tau, mu), 0.7, atol=1e-14)
    rng = np.random.default_rng(1)
    M, N = 8, 12
    F = rng.standard_normal((M, N))
    T1 = np.eye(M) - 2 * tau * mu * neumann_A(M)
    T2 = np.eye(N) - 2 * tau * mu * neumann_A(N)
    ref = 0.5 * (np.linalg.solve(T1, F) + np.linalg.solve(T2, F.T).T)
    assert np.max(np.abs(orc.solve_aos(F, tau, mu) - ref)) < 1e-13


def test_aos_consistent_with_exact_neumann_solve(orc):
    """AOS = (1 - tau mu Delta)^{-1} + O((tau mu)^2): halving tau mu cuts the difference ~4x."""
    M = N = 32
    ii, jj = np.meshgrid(np.arange(M), np.arange(N), indexing="ij")
    F = np.cos(np.pi * ii / (M - 1)) * np.cos(2 * np.pi * jj / (N - 1)) + 0.3
    lap = np.kron(neumann_A(M), np.eye(N)) + np.kron(np.eye(M), neumann_A(N))
    errs = []
    for tm in (0.1, 0.05, 0.025):
        exact = np.linalg.solve(np.eye(M * N) - tm * lap, F.ravel()).reshape(M, N)
        errs.append(np.max(np.abs(orc.solve_aos(F, tm, 1.0) - exact)))
    assert errs[1] < errs[0] / 3 and errs[2] < errs[1] / 3.5    # ratio -> 4 (second order)
