"""Pin of the oracle's phi right-hand side, Eq. (37), against the energy it descends.

The discrete sub-problem energy (Eq. 22 with w = w^k, b = b^k fixed, Eq. 24) is

  E1(psi) = sum_x [gamma g |w| delta(psi) + alpha g (1 - H(psi))]
            - beta sum_x sum_{y in W(x)} G(x - y) w(x).w(y) h(psi(x)) h(psi(y))
            + mu/2 sum_x |w - grad psi - b|^2 .

Eq. (26)/(30) treat mu Delta psi implicitly and everything else explicitly, so
(F - psi)/tau = -dE1/dpsi - mu div(grad psi).  The gradient is taken by
central finite differences of E1 (SPEC acceptance criterion 8): a
dropped term, a wrong sign, a missing factor 2 or a transposed div fails it.
"""
import numpy as np
import pytest


def disc(R, shape):
    return [(p, q) for p in range(-R, R + 1) for q in range(-R, R + 1) if shape == 1 or p * p + q * q <= R * R]


def energy(orc, P, psi, w1, w2, b1, b2, g):
    eps, l = P["epsilon"], P["l"]
    M, N = psi.shape
    dl = np.vectorize(lambda x: orc.delta(x, eps))(psi)
    Hv = np.vectorize(lambda x: orc.H(x, eps))(psi)
    hv = np.vectorize(lambda x: orc.h(x, eps, l))(psi)
    wn = np.sqrt(w1 ** 2 + w2 ** 2)
    E = np.sum(P["gamma"] * g * wn * dl + P["alpha"] * g * (1 - Hv))
    R, d = P["window"], P["d"]
    Er = 0.0
    for i in range(M):
        for j in range(N):
            for p, q in disc(R, P["window_shape"]):
                y = (i + p, j + q)
                if 0 <= y[0] < M and 0 <= y[1] < N:
                    G = np.exp(-(p * p + q * q) / d ** 2)
                    Er += G * (w1[i, j] * w1[y] + w2[i, j] * w2[y]) * hv[i, j] * hv[y]
    E -= P["beta"] * Er
    gp1, gp2 = orc.grad(psi)
    E += P["mu"] / 2 * np.sum((w1 - gp1 - b1) ** 2 + (w2 - gp2 - b2) ** 2)
    return E


@pytest.mark.parametrize("eps,l,shape", [(0.5, 0.5, 0), (1.0, 1.0, 0), (0.7, 0.4, 1)])
def test_rhs_is_descent_direction_of_E1(orc, eps, l, shape):
    from synth import paper_params
    P = paper_params(2, epsilon=eps, l=l, window_shape=shape, d=1.7)
    rng = np.random.default_rng(17)
    M, N = 7, 8
    psi = rng.uniform(-(l + eps), l + eps, (M, N))
    w1, w2 = rng.uniform(-1, 1, (M, N)), rng.uniform(-1, 1, (M, N))
    b1, b2 = 0.3 * rng.standard_normal((M, N)), 0.3 * rng.standard_normal((M, N))
    g = rng.uniform(0.1, 1.0, (M, N))
    F = orc.rhs(P, psi, w1, w2, b1, b2, g)
    lap = orc.div(*orc.grad(psi))
    hstep = 1e-6
    for i in range(M):
        for j in range(N):
            e = np.zeros((M, N))
            e[i, j] = hstep
            dE = (energy(orc, P, psi + e, w1, w2, b1, b2, g) - energy(orc, P, psi - e, w1, w2, b1, b2, g)) / (2 * hstep)
            lhs = (F[i, j] - psi[i, j]) / P["tau"]
            rhs = -dE - P["mu"] * lap[i, j]
            assert lhs == pytest.approx(rhs, rel=1e-6, abs=1e-6 * (1 + abs(rhs)))


def test_rhs_tau_zero_is_identity(orc):
    from synth import paper_params
    rng = np.random.default_rng(2)
    P = paper_params(3, tau=0.0)
    psi = rng.uniform(-1, 1, (9, 9))
    z = rng.uniform(-1, 1, (9, 9))
    assert np.array_equal(orc.rhs(P, psi, z, z, z, z, np.abs(z)), psi)
