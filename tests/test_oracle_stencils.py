"""Pins of the oracle's discrete gradient / divergence (Eq. 35, 36; reading Q6)."""
import numpy as np


def test_adjointness(orc):
    """<grad phi, u> = -<phi, div u> for every phi, u."""
    rng = np.random.default_rng(1)
    for M, N in ((4, 4), (5, 7), (1, 6), (8, 1)):
        phi = rng.standard_normal((M, N))
        u1, u2 = rng.standard_normal((M, N)), rng.standard_normal((M, N))
        g1, g2 = orc.grad(phi)
        lhs = np.sum(g1 * u1 + g2 * u2)
        rhs = -np.sum(phi * orc.div(u1, u2))
        assert abs(lhs - rhs) < 1e-12


def test_grad_constant_and_linear(orc):
    g1, g2 = orc.grad(np.full((3, 3), 5.0))
    assert not g1.any() and not g2.any()
    ii = np.tile(np.arange(6.0)[:, None], (1, 5))
    g1, g2 = orc.grad(ii)
    assert np.all(g1[:-1] == 1.0) and np.all(g1[-1] == 0.0) and not g2.any()


def test_div_grad_is_neumann_laplacian(orc):
    """div(grad phi) = 5-point Laplacian of Eq. (35) with replicated (Neumann) ghost values."""
    rng = np.random.default_rng(2)
    phi = rng.standard_normal((6, 7))
    lap = orc.div(*orc.grad(phi))
    p = np.pad(phi, 1, mode="edge")
    ref = p[:-2, 1:-1] + p[2:, 1:-1] + p[1:-1, :-2] + p[1:-1, 2:] - 4 * phi
    assert np.allclose(lap, ref, atol=1e-13)


def test_quadratic_field(orc):
    """phi = i^2 -> Laplacian 2 at interior rows."""
    phi = np.tile((np.arange(8.0) ** 2)[:, None], (1, 5))
    lap = orc.div(*orc.grad(phi))
    assert np.allclose(lap[1:-1], 2.0)
