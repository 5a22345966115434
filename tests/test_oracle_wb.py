"""Pins of the oracle's w sub-problem: shrink (Eq. 42), projection (Eq. 40), w/b update (Eq. 41, 23)
and the fixed-point variant (Eq. 38-39)."""
import numpy as np
import pytest


def test_shrink_closed_forms(orc):
    assert orc.shrink(2.0, 0.0, 1.0) == pytest.approx((1.0, 0.0))
    assert orc.shrink(3.0, 4.0, 1.0) == pytest.approx((2.4, 3.2))
    assert orc.shrink(0.3, 0.4, 0.5) == (0.0, 0.0)                           # |B| <= t
    assert orc.shrink(0.3, 0.4, 0.0) == pytest.approx((0.3, 0.4))            # t = 0
    assert orc.shrink(0.0, 0.0, 0.0) == (0.0, 0.0)                           # 0 * 0/|0| = 0, Eq. (42)


def test_shrink_minimizes_by_brute_force(orc):
    """Eq. (42) is the minimizer of t|w| + 1/2 |w - B|^2 (the pointwise w energy of Eq. 22)."""
    rng = np.random.default_rng(4)
    xs = np.linspace(-3, 3, 1201)
    X, Y = np.meshgrid(xs, xs, indexing="ij")
    for _ in range(10):
        B = rng.uniform(-2, 2, 2)
        t = rng.uniform(0, 1.5)
        J = t * np.hypot(X, Y) + 0.5 * ((X - B[0]) ** 2 + (Y - B[1]) ** 2)
        k = np.unravel_index(np.argmin(J), J.shape)
        w = orc.shrink(B[0], B[1], t)
        assert abs(w[0] - X[k]) <= 0.01 and abs(w[1] - Y[k]) <= 0.01


def test_projection_modes(orc):
    assert orc.project(0, 2.4, 3.2) == pytest.approx((0.6, 0.8))      # |w~| = 4
    assert orc.project(0, 0.3, 0.4) == (0.3, 0.4)                    # inside the ball: identity
    a = orc.project(0, 5.0, -1.0)
    assert orc.project(0, *a) == pytest.approx(a)                     # idempotent
    assert orc.project(1, 0.3, 0.4) == pytest.approx((0.6, 0.8))      # Eq. (40) sphere
    assert orc.project(1, 0.0, 0.0) == (0.0, 0.0)
    assert orc.project(2, 3.0, 4.0) == (3.0, 4.0)


def test_ball_projection_is_nearest_point(orc):
    rng = np.random.default_rng(9)
    ang = np.linspace(0, 2 * np.pi, 20001)
    for _ in range(5):
        a = rng.uniform(-3, 3, 2)
        p = orc.project(0, *a)
        if np.hypot(*a) > 1:
            dist = np.hypot(np.cos(ang) - a[0], np.sin(ang) - a[1])
            k = np.argmin(dist)
            assert abs(p[0] - np.cos(ang[k])) < 1e-3 and abs(p[1] - np.sin(ang[k])) < 1e-3


def _state(rng, M, N):
    phi = rng.uniform(-1, 1, (M, N))
    return dict(phi=phi, w1=rng.uniform(-1, 1, (M, N)), w2=rng.uniform(-1, 1, (M, N)),
                b1=0.2 * rng.standard_normal((M, N)), b2=0.2 * rng.standard_normal((M, N)),
                g=rng.uniform(0.1, 1, (M, N)))


def test_wb_bregman_identity_and_ball(orc):
    """b^{k+1} - b^k = grad phi - w^{k+1} exactly (Eq. 23); |w^{k+1}| <= 1 under BALL."""
    from synth import paper_params
    rng = np.random.default_rng(10)
    s = _state(rng, 12, 10)
    P = paper_params(3)
    w1, w2, b1, b2 = orc.wb(P, s["phi"], s["w1"], s["w2"], s["b1"], s["b2"], s["g"])
    g1, g2 = orc.grad(s["phi"])
    assert np.allclose(b1 - s["b1"], g1 - w1, atol=1e-15)
    assert np.allclose(b2 - s["b2"], g2 - w2, atol=1e-15)
    assert np.all(np.hypot(w1, w2) <= 1 + 1e-15)


def test_wb_reduces_to_shrink_without_repulsion(orc):
    """beta = 0: w = shrink(grad phi + b, (gamma/mu) g delta(phi)) pixel by pixel (NONE projection)."""
    from synth import paper_params
    rng = np.random.default_rng(12)
    s = _state(rng, 6, 7)
    P = paper_params(2, beta=0.0, w_proj=2)
    w1, w2, _, _ = orc.wb(P, s["phi"], s["w1"], s["w2"], s["b1"], s["b2"], s["g"])
    g1, g2 = orc.grad(s["phi"])
    for i in range(6):
        for j in range(7):
            t = P["gamma"] / P["mu"] * s["g"][i, j] * orc.delta(s["phi"][i, j], P["epsilon"])
            e = orc.shrink(g1[i, j] + s["b1"][i, j], g2[i, j] + s["b2"][i, j], t)
            assert (w1[i, j], w2[i, j]) == pytest.approx(e, abs=1e-15)


def test_wb_repulsion_term_by_impulse(orc):
    """One non-zero w at c, phi = 0 (h = 1, delta = 2 for eps=1/2), gamma = 0 (t = 0), NONE projection:
    B(x) = grad phi + b + (2 beta/mu) G(x - c) w_c  (Eq. 41)."""
    from synth import paper_params
    P = paper_params(3, gamma=0.0, w_proj=2)
    M = N = 11
    z = np.zeros((M, N))
    w1 = z.copy()
    w1[5, 5] = 1.0
    n1, n2, _, _ = orc.wb(P, z, w1, z, z, z, np.ones((M, N)))
    for i in range(M):
        for j in range(N):
            r2 = (i - 5) ** 2 + (j - 5) ** 2
            G = np.exp(-r2 / 9.0) if r2 <= 9 else 0.0
            assert n1[i, j] == pytest.approx(2 * P["beta"] / P["mu"] * G, abs=1e-15)
            assert n2[i, j] == 0.0


def test_b_telescoping(orc):
    """b^K = sum_k (grad phi^k - w^k) over the iterations."""
    from synth import paper_params
    rng = np.random.default_rng(13)
    s = _state(rng, 8, 8)
    P = paper_params(2)
    w1, w2, b1, b2 = s["w1"], s["w2"], np.zeros((8, 8)), np.zeros((8, 8))
    acc1, acc2 = np.zeros((8, 8)), np.zeros((8, 8))
    for k in range(4):
        phi = np.clip(s["phi"] + 0.1 * k * rng.standard_normal((8, 8)), -1, 1)
        w1, w2, b1, b2 = orc.wb(P, phi, w1, w2, b1, b2, s["g"])
        g1, g2 = orc.grad(phi)
        acc1 += g1 - w1
        acc2 += g2 - w2
    assert np.allclose(b1, acc1, atol=1e-14) and np.allclose(b2, acc2, atol=1e-14)


def test_fixed_point_mode(orc):
    """Eq. (39) with one sweep: w = proj((mu grad phi + mu b + 2 beta h v)/(gamma g delta + mu)).
    With beta = 0 it is (grad phi + b) mu/(gamma g delta + mu) per pixel."""
    from synth import paper_params
    rng = np.random.default_rng(14)
    s = _state(rng, 6, 6)
    P = paper_params(2, beta=0.0, w_mode=1, w_iters=1, w_proj=2)
    w1, w2, _, _ = orc.wb(P, s["phi"], s["w1"], s["w2"], s["b1"], s["b2"], s["g"])
    g1, g2 = orc.grad(s["phi"])
    for i in range(6):
        for j in range(6):
            den = P["gamma"] * s["g"][i, j] * orc.delta(s["phi"][i, j], P["epsilon"]) + P["mu"]
            assert w1[i, j] == pytest.approx(P["mu"] * (g1[i, j] + s["b1"][i, j]) / den, abs=1e-14)
            assert w2[i, j] == pytest.approx(P["mu"] * (g2[i, j] + s["b2"][i, j]) / den, abs=1e-14)


def _fixed_point_reference(orc, P, phi, w1, w2, b1, b2, g, passes):
    """Eq. (38)-(39) written out pass by pass from pinned pieces (orc.grad: Eq. 35; orc.h: Eq. 11;
    orc.window_sum: P:368, pinned by impulse / full-window / locality in test_oracle_window.py):
    w^{k+1,0} = w^k and, for r = 0..passes-1,
        v^r    = sum_W G h(phi^{k+1}) w^{k+1,r}                           (Eq. 38)
        w^{r+1} = (mu grad phi + mu b + 2 beta h v^r) / (gamma g delta + mu)   (Eq. 39)
    with the NONE projection (Q1)."""
    eps, l = P["epsilon"], P["l"]
    hv = np.vectorize(lambda x: orc.h(x, eps, l))(phi)
    dl = np.vectorize(lambda x: orc.delta(x, eps))(phi)
    gp1, gp2 = orc.grad(phi)
    n1, n2 = w1.copy(), w2.copy()
    for _ in range(passes):
        v1, v2 = orc.window_sum(hv * n1, hv * n2, P["window"], P["d"], P["window_shape"])
        den = P["gamma"] * g * dl + P["mu"]
        n1 = (P["mu"] * gp1 + P["mu"] * b1 + 2 * P["beta"] * hv * v1) / den
        n2 = (P["mu"] * gp2 + P["mu"] * b2 + 2 * P["beta"] * hv * v2) / den
    return n1, n2


@pytest.mark.parametrize("passes", [1, 2, 3])
def test_fixed_point_passes_recompute_v_from_the_previous_pass(orc, passes):
    """NEXT-2 pin with beta != 0 and several passes: one impulse of w^k at the centre, phi = 0 where
    h(0) = 1, gamma = 0.  Pass r+1 must use v^r built from w^{k+1,r} (Eq. 38), not from w^k: with the
    impulse the two readings differ from the second pass on (the first pass spreads the impulse over
    the window, the second spreads that again).  Also the gamma != 0 denominator on a random state."""
    from synth import paper_params
    M, N = 15, 13
    phi = np.zeros((M, N))
    w1, w2 = np.zeros((M, N)), np.zeros((M, N))
    w1[7, 6], w2[7, 6] = 0.8, -0.5
    b1, b2 = np.zeros((M, N)), np.zeros((M, N))
    g = np.ones((M, N))
    P = paper_params(3, gamma=0.0, beta=0.6, w_mode=1, w_iters=passes, w_proj=2)
    n1, n2, nb1, nb2 = orc.wb(P, phi, w1, w2, b1, b2, g)
    r1, r2 = _fixed_point_reference(orc, P, phi, w1, w2, b1, b2, g, passes)
    assert np.allclose(n1, r1, atol=1e-14) and np.allclose(n2, r2, atol=1e-14)
    gp1, gp2 = orc.grad(phi)
    assert np.allclose(nb1, b1 + gp1 - n1, atol=1e-15) and np.allclose(nb2, b2 + gp2 - n2, atol=1e-15)
    if passes >= 2:
        # the reading "v^r from w^k" would give the one-pass result at every pass: it must differ
        s1, s2 = _fixed_point_reference(orc, P, phi, w1, w2, b1, b2, g, 1)
        assert np.max(np.abs(n1 - s1)) > 1e-3
        # a pixel two window radii from the impulse: zero after one pass, reached only through w^{k+1,1}
        assert s1[7, 12] == 0.0 and s1[7, 9] != 0.0
        assert abs(n1[7, 12]) > 1e-6
    # random state, gamma != 0, through the same reference
    rng = np.random.default_rng(33)
    s = _state(rng, 9, 11)
    P = paper_params(2, beta=0.4, w_mode=1, w_iters=passes, w_proj=2)
    n1, n2, _, _ = orc.wb(P, s["phi"], s["w1"], s["w2"], s["b1"], s["b2"], s["g"])
    r1, r2 = _fixed_point_reference(orc, P, s["phi"], s["w1"], s["w2"], s["b1"], s["b2"], s["g"], passes)
    assert np.allclose(n1, r1, atol=1e-13) and np.allclose(n2, r2, atol=1e-13)
