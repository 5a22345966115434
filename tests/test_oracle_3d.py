"""Pins of the 3-D oracle (NEXT-3, reading Q26: every operator of the 2-D method gains the depth
axis).  Nothing here re-types the oracle's formulas:

  * a D = 1 volume must reproduce the (independently pinned) 2-D oracle functions exactly --
    a dropped or mis-indexed in-plane term fails it;
  * the 3-D FFT against numpy.fft.fftn and a brute-force DFT, the 3-D solve against a dense
    numpy.linalg.solve of the periodic 7-point system and its residual;
  * grad / div adjointness and div(grad) of a quadratic (closed form 6 in the interior);
  * the ball window by its impulse response and by a constant field (closed-form weight sum);
  * the RHS against the finite-difference gradient of the 3-D sub-problem energy E1 (a wrong
    sign, factor or axis in any term fails it);
  * shrink / projection closed forms on 3-vectors; plateau fixed point and the clamp.
"""
import itertools

import numpy as np
import pytest


def _p(window=2, **over):
    from synth import paper_params
    p = paper_params(window)
    p.update(over)
    return p


def _rand(shape, seed, lo=-1.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, shape)


# ----------------------------------------------------------------------------- D = 1 reduces to 2-D
def test_d1_reduces_to_2d(orc):
    M, N = 12, 16
    P = _p(3, d=2.5)
    psi = _rand((1, M, N), 1, -1.4, 1.4)
    w = [_rand((1, M, N), 2), _rand((1, M, N), 3), np.zeros((1, M, N))]
    b = [0.3 * _rand((1, M, N), 4), 0.3 * _rand((1, M, N), 5), np.zeros((1, M, N))]
    g = _rand((1, M, N), 6, 0.1, 1.0)
    # gradient / divergence
    g3 = orc.grad3(psi)
    g2 = orc.grad(psi[0])
    assert np.array_equal(g3[0][0], g2[0]) and np.array_equal(g3[1][0], g2[1]) and not g3[2].any()
    assert np.array_equal(orc.div3(w[0], w[1], w[2])[0], orc.div(w[0][0], w[1][0]))
    # window
    v3 = orc.window_sum3(w[0], w[1], w[2], 3, 2.5, 0)
    v2 = orc.window_sum(w[0][0], w[1][0], 3, 2.5, 0)
    assert np.allclose(v3[0][0], v2[0], atol=1e-14) and np.allclose(v3[1][0], v2[1], atol=1e-14)
    # RHS, solve, w/b update, edge indicator
    F3 = orc.rhs3(P, psi, w, b, g)
    F2 = orc.rhs(P, psi[0], w[0][0], w[1][0], b[0][0], b[1][0], g[0])
    assert np.allclose(F3[0], F2, rtol=1e-13, atol=1e-13)
    assert np.allclose(orc.solve3(F3, P["tau"], P["mu"])[0], orc.solve(F2, P["tau"], P["mu"]), atol=1e-12)
    (nw, nb) = orc.wb3(P, psi, w, b, g)
    r1, r2, rb1, rb2 = orc.wb(P, psi[0], w[0][0], w[1][0], b[0][0], b[1][0], g[0])
    for a, r in ((nw[0][0], r1), (nw[1][0], r2), (nb[0][0], rb1), (nb[1][0], rb2)):
        assert np.allclose(a, r, atol=1e-13)
    assert not nw[2].any() and not nb[2].any()
    img = _rand((1, M, N), 7, 0, 1)
    assert np.allclose(orc.edge3(img, 1.0, 30.0, 2)[0], orc.edge(img[0], 1.0, 30.0, 2), atol=1e-13)


def test_d1_trajectory_matches_2d(orc):
    from synth import make_config
    c = make_config("c1")
    p = c["params"]
    st2 = orc.run(p, c["image"][0], c["phi0"][0], 3)
    st3 = orc.run3(p, c["image"][:1], c["phi0"][:1], 3)
    assert np.allclose(st3["phi"][0], st2["phi"], atol=1e-11)


# ----------------------------------------------------------------------------- FFT and solve
def test_fft3_matches_numpy_and_bruteforce(orc):
    x = _rand((4, 2, 8), 8) + 1j * _rand((4, 2, 8), 9)
    X = orc.fft3(x)
    assert np.allclose(X, np.fft.fftn(x), atol=1e-12)
    D, M, N = x.shape
    k = (1, 1, 5)
    brute = sum(x[z, i, j] * np.exp(-2j * np.pi * (k[0] * z / D + k[1] * i / M + k[2] * j / N))
                for z, i, j in itertools.product(range(D), range(M), range(N)))
    assert abs(X[k] - brute) < 1e-12
    assert np.allclose(orc.fft3(X, inverse=True), x, atol=1e-13)


def _periodic_laplacian3(phi):
    return sum(np.roll(phi, s, a) for a in range(3) for s in (1, -1)) - 6 * phi


def test_solve3_dense_and_residual(orc):
    tau, mu = 0.05, 8.0
    D, M, N = 4, 4, 4
    n = D * M * N
    A = np.zeros((n, n))
    for q in range(n):
        e = np.zeros(n)
        e[q] = 1
        A[:, q] = (e.reshape(D, M, N) - tau * mu * _periodic_laplacian3(e.reshape(D, M, N))).ravel()
    F = _rand((D, M, N), 10)
    ref = np.linalg.solve(A, F.ravel()).reshape(D, M, N)
    assert np.allclose(orc.solve3(F, tau, mu), ref, atol=1e-12)
    F = _rand((8, 16, 8), 11)
    for tm in (0.1, 0.8, 5.0):
        phi = orc.solve3(F, 1.0, tm)
        res = np.linalg.norm(phi - tm * _periodic_laplacian3(phi) - F) / np.linalg.norm(F)
        assert res < 1e-10
    assert orc.symbol3(8, 8, 8, tau, mu, 0, 0, 0) == 1.0
    assert orc.symbol3(8, 8, 8, tau, mu, 4, 4, 4) == pytest.approx(1 + 12 * tau * mu)


# ----------------------------------------------------------------------------- stencils
def test_grad3_div3_adjoint_and_laplacian(orc):
    phi = _rand((5, 6, 7), 12)
    u = [_rand((5, 6, 7), 13 + c) for c in range(3)]
    lhs = sum(np.sum(a * b) for a, b in zip(orc.grad3(phi), u))
    rhs = -np.sum(phi * orc.div3(*u))
    assert lhs == pytest.approx(rhs, rel=1e-12)
    z, i, j = np.meshgrid(np.arange(6.0), np.arange(7.0), np.arange(8.0), indexing="ij")
    lap = orc.div3(*orc.grad3(z ** 2 + i ** 2 + j ** 2))
    assert np.allclose(lap[1:-1, 1:-1, 1:-1], 6.0, atol=1e-12)


def test_window_sum3_impulse_and_constant(orc):
    R, d = 2, 1.5
    D = M = N = 9
    u = np.zeros((D, M, N))
    u[4, 4, 4] = 1.0
    v, _, _ = orc.window_sum3(u, 0 * u, 0 * u, R, d, 0)
    for z, i, j in itertools.product(range(D), range(M), range(N)):
        r2 = (z - 4) ** 2 + (i - 4) ** 2 + (j - 4) ** 2
        expect = np.exp(-r2 / d ** 2) if r2 <= R * R else 0.0
        assert v[z, i, j] == pytest.approx(expect, abs=1e-15)
    ones = np.ones((D, M, N))
    v, _, _ = orc.window_sum3(ones, ones, ones, R, d, 0)
    ball = sum(np.exp(-(p * p + q * q + r * r) / d ** 2) for p, q, r in itertools.product(range(-R, R + 1), repeat=3)
               if p * p + q * q + r * r <= R * R)
    assert v[4, 4, 4] == pytest.approx(ball, rel=1e-14)
    cube = sum(np.exp(-(p * p + q * q + r * r) / d ** 2) for p, q, r in itertools.product(range(-R, R + 1), repeat=3))
    v, _, _ = orc.window_sum3(ones, ones, ones, R, d, 1)
    assert v[4, 4, 4] == pytest.approx(cube, rel=1e-14)


# ----------------------------------------------------------------------------- RHS = -grad E1 (3-D)
def _energy3(orc, P, psi, w, b, g):
    eps, l = P["epsilon"], P["l"]
    dl = np.vectorize(lambda x: orc.delta(x, eps))(psi)
    Hv = np.vectorize(lambda x: orc.H(x, eps))(psi)
    hv = np.vectorize(lambda x: orc.h(x, eps, l))(psi)
    wn = np.sqrt(sum(a ** 2 for a in w))
    E = np.sum(P["gamma"] * g * wn * dl + P["alpha"] * g * (1 - Hv))
    R, d = P["window"], P["d"]
    D, M, N = psi.shape
    Er = 0.0
    for x in itertools.product(range(D), range(M), range(N)):
        for r, p, q in itertools.product(range(-R, R + 1), repeat=3):
            if p * p + q * q + r * r > R * R:
                continue
            y = (x[0] + r, x[1] + p, x[2] + q)
            if 0 <= y[0] < D and 0 <= y[1] < M and 0 <= y[2] < N:
                G = np.exp(-(p * p + q * q + r * r) / d ** 2)
                Er += G * sum(a[x] * a[y] for a in w) * hv[x] * hv[y]
    E -= P["beta"] * Er
    gp = orc.grad3(psi)
    E += P["mu"] / 2 * sum(np.sum((w[c] - gp[c] - b[c]) ** 2) for c in range(3))
    return E


def test_rhs3_is_descent_direction_of_E1(orc):
    P = _p(1, epsilon=0.5, l=0.5, d=1.3)
    shape = (3, 4, 4)
    psi = _rand(shape, 20, -1.0, 1.0)
    w = [_rand(shape, 21 + c) for c in range(3)]
    b = [0.3 * _rand(shape, 24 + c) for c in range(3)]
    g = _rand(shape, 27, 0.1, 1.0)
    F = orc.rhs3(P, psi, w, b, g)
    lap = orc.div3(*orc.grad3(psi))
    h = 1e-6
    for x in itertools.product(*[range(s) for s in shape]):
        e = np.zeros(shape)
        e[x] = h
        dE = (_energy3(orc, P, psi + e, w, b, g) - _energy3(orc, P, psi - e, w, b, g)) / (2 * h)
        lhs = (F[x] - psi[x]) / P["tau"]
        assert lhs == pytest.approx(-dE - P["mu"] * lap[x], rel=1e-6, abs=1e-6 * (1 + abs(dE)))


# ----------------------------------------------------------------------------- w / b and the iteration
def test_shrink3_project3_closed_forms(orc):
    assert np.allclose(orc.shrink3([2.0, 0.0, 0.0], 1.0), [1, 0, 0])
    assert np.allclose(orc.shrink3([2.0, 3.0, 6.0], 2.0), np.array([2.0, 3.0, 6.0]) * 5 / 7)   # |B| = 7
    assert not orc.shrink3([0.1, 0.1, 0.1], 1.0).any()
    assert np.allclose(orc.shrink3([0.3, -0.2, 0.5], 0.0), [0.3, -0.2, 0.5])
    assert np.allclose(orc.project3(0, [2.0, 3.0, 6.0]), np.array([2.0, 3.0, 6.0]) / 7)
    assert np.allclose(orc.project3(0, [0.2, 0.1, 0.3]), [0.2, 0.1, 0.3])
    assert np.allclose(orc.project3(1, [0.2, 0.1, 0.2]), np.array([0.2, 0.1, 0.2]) / 0.3)


def test_plateau_fixed_point_and_clamp(orc):
    P = _p(2)
    shape = (4, 8, 8)
    st = {"phi": np.ones(shape), "w": tuple(np.zeros(shape) for _ in range(3)),
          "b": tuple(np.zeros(shape) for _ in range(3))}
    orc.iterate3(P, st, np.ones(shape), 2)
    assert np.allclose(st["phi"], 1.0, atol=1e-12)
    phi0 = np.where(_rand(shape, 30) > 0, 1.0, -1.0)
    st = orc.init3(phi0)
    orc.iterate3(P, st, _rand(shape, 31, 0.2, 1.0), 2)
    assert np.abs(st["phi"]).max() <= 1.0


# ----------------------------------------------------------------------------- depth axis and third channel
def test_edge3_matches_scipy_gaussian_and_central_differences(orc):
    """Eq. (1) in 3-D (Q16, Q26) against an independent library pipeline: scipy's separable
    normalized Gaussian with replicate padding (mode="nearest", truncate=3 -> radius ceil(3 sigma)),
    then central differences with replicate padding along all three axes."""
    from scipy import ndimage
    f = _rand((7, 9, 10), 40, 0.0, 1.0)
    f[2:5, 3:7, 4:8] += 1.0                       # a block edge along every axis, incl. depth
    for rho, s in ((30.0, 2), (5.0, 1)):
        fs = ndimage.gaussian_filter(f, sigma=1.0, mode="nearest", truncate=3.0)
        p = np.pad(fs, 1, mode="edge")
        gz = (p[2:, 1:-1, 1:-1] - p[:-2, 1:-1, 1:-1]) / 2
        gi = (p[1:-1, 2:, 1:-1] - p[1:-1, :-2, 1:-1]) / 2
        gj = (p[1:-1, 1:-1, 2:] - p[1:-1, 1:-1, :-2]) / 2
        m2 = gz ** 2 + gi ** 2 + gj ** 2
        ref = 1.0 / (1.0 + rho * (m2 if s == 2 else np.sqrt(m2)))
        assert np.allclose(orc.edge3(f, 1.0, rho, s), ref, rtol=0, atol=1e-12)
        assert np.abs(gz).max() > 0.1               # the depth axis carries real signal


_COMP_OF_AXIS = {1: 0, 2: 1, 0: 2}                 # array axis (z, i, j) -> component (1, 2, 3) = (i, j, z)


def _perm_field(a, perm):
    return np.ascontiguousarray(np.transpose(a, perm))


def _perm_vec(v, perm):
    """Permute a 3-vector field: new component along new axis a = old component along old axis perm[a]."""
    out = [None, None, None]
    for a in range(3):
        out[_COMP_OF_AXIS[a]] = _perm_field(v[_COMP_OF_AXIS[perm[a]]], perm)
    return tuple(out)


@pytest.mark.parametrize("perm", [(0, 2, 1), (1, 0, 2), (2, 1, 0), (1, 2, 0)])
def test_axis_permutation_commutes_with_every_3d_function(orc, perm):
    """Metamorphic pin of the depth axis and the third channel (Q26: the 3-D operators are the 2-D
    ones with an identical third axis): on a D = M = N cube, permuting the axes (and the vector
    components with them) commutes with grad, div, the edge indicator, the ball / cube window sum,
    the periodic solve, the RHS, the w/b update (threshold and fixed-point, BALL) and a full
    iteration.  A wrong index, sign or weight on any one axis or channel breaks the symmetry."""
    n = 6
    sh = (n, n, n)
    P = _p(2, d=1.7, beta=0.5)
    psi = _rand(sh, 50, -1.2, 1.2)
    w = tuple(_rand(sh, 51 + c) for c in range(3))
    b = tuple(0.3 * _rand(sh, 54 + c) for c in range(3))
    g = _rand(sh, 57, 0.1, 1.0)
    pf = lambda a: _perm_field(a, perm)                                   # noqa: E731
    pv = lambda v: _perm_vec(v, perm)                                     # noqa: E731
    close = lambda a, r: np.allclose(a, r, rtol=0, atol=1e-12)            # noqa: E731
    # grad / div
    assert all(close(a, r) for a, r in zip(orc.grad3(pf(psi)), pv(orc.grad3(psi))))
    assert close(orc.div3(*pv(w)), pf(orc.div3(*w)))
    # edge indicator
    img = _rand(sh, 58, 0.0, 1.0)
    assert close(orc.edge3(pf(img), 1.0, 30.0, 2), pf(orc.edge3(img, 1.0, 30.0, 2)))
    # window sums (ball and cube)
    for shape in (0, 1):
        assert all(close(a, r) for a, r in zip(orc.window_sum3(*pv(w), 2, 1.7, shape),
                                               pv(orc.window_sum3(*w, 2, 1.7, shape))))
    # solve (the 3-D symbol is symmetric in the axes when D = M = N)
    F = _rand(sh, 59)
    assert close(orc.solve3(pf(F), P["tau"], P["mu"]), pf(orc.solve3(F, P["tau"], P["mu"])))
    # RHS
    assert close(orc.rhs3(P, pf(psi), pv(w), pv(b), pf(g)), pf(orc.rhs3(P, psi, w, b, g)))
    # w/b update, both modes
    for over in (dict(), dict(w_mode=1, w_iters=2)):
        Q = dict(P, **over)
        nw, nb = orc.wb3(Q, pf(psi), pv(w), pv(b), pf(g))
        rw, rb = orc.wb3(Q, psi, w, b, g)
        assert all(close(a, r) for a, r in zip(nw + nb, pv(rw) + pv(rb)))
    # one full iteration
    st = {"phi": psi.copy(), "w": w, "b": b}
    sp = {"phi": pf(psi), "w": pv(w), "b": pv(b)}
    orc.iterate3(P, st, g, 1)
    orc.iterate3(P, sp, pf(g), 1)
    assert close(sp["phi"], pf(st["phi"]))
    assert all(close(a, r) for a, r in zip(sp["w"] + sp["b"], pv(st["w"]) + pv(st["b"])))
