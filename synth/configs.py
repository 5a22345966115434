"""Synthetic stand-ins for the paper's images (BASELINE.json `configs`).

The paper's own images (two circles, hand, cells, grains, CT; §5,
P:434-574) are not available, so every workload is generated here from a seed
with numpy's PCG64.  The recipe is stated per config in DESIGN.md §3.

Conventions
-----------
* Arrays are float32, shape [B][M][N], row-major, i = row, j = column.
* BASELINE.json writes the initial level set as "+1 inside".  The paper puts
  phi < 0 inside (Eq. 3).  The two are equivalent under phi -> -phi
  (reading R-sign).  `make_config` returns `phi0` in the PAPER's
  convention (already negated), which is what the oracle and the library take.
* Noise is added last and is not clipped.

Nothing here implements any step of the Split Bregman method; the only image
processing is the "thresholded smoothed image" initialisation of C4, which is
part of the input recipe (BASELINE.json configs[3]), done with scipy.ndimage.
"""
from __future__ import annotations

import math

import numpy as np

BASE_SEED = 12693


def paper_params(window: int, **over) -> dict:
    """Parameter set used for every config (readings Q17, Q22, Q23).

    From the Fig. 1 caption: alpha=4, beta=0.2, mu=8, S=3.  d = window radius
    (Eq. 38 ties the half-width to d, reading Q2); s=2, sigma=1 (north_star's
    g = 1/(1+|grad(G_sigma*I)|^2)); phi clamped to [-1, 1] (north_star); w projected onto the
    unit ball (reading Q1); disc window.
    Q22: epsilon = l = 1/2 -- with the clamp, the caption's epsilon = l = 1 put the +-1 plateaus
         on the band edge and every C1 contour collapses in the oracle.
    Q23: gamma = 1, tau = 0.05 -- the explicit -gamma g |w| delta'(phi) term of Eq. (37) has
         pointwise stiffness tau gamma pi^2 / (2 eps^3); with eps = 1/2 the caption's gamma = 4,
         tau = 0.1 give 15.8 and the fp64 oracle itself amplifies a 1e-7 perturbation to O(1)
         in 10 iterations; gamma = 1, tau = 0.05 give 1.97 (the caption set's own value at eps = 1).
    Q24: beta = 0.2 * G5 / G_W(window, d), G_W = sum over the window of exp(-(p^2+q^2)/d^2) and
         G5 = 21.4 the same sum for the caption's 5x5 window with d = 5: the repulsion
         strength beta * G_W stays the caption's ("an excessively large beta causes the
         contour to become unstable"); without it the R = 6 config amplifies 1e-6 to 0.1 in 10
         iterations of the fp64 oracle.
    rho = 30 (unstated in the paper, reading Q4): C1 keeps one component.
    """
    d = float(over.get("d", window if window > 0 else 1.0))
    shape = int(over.get("window_shape", 0))
    p = dict(gamma=1.0, alpha=4.0, beta=repulsion_beta(window, d, shape), mu=8.0, epsilon=0.5, l=0.5,
             d=d, window=int(window), window_shape=shape, tau=0.05, S=3,
             rho=30.0, sigma=1.0, s=2, phi_clip=1.0, w_proj=0, w_mode=0, w_iters=1, phi_solver=0)
    p.update(over)
    return p


def window_weight_sum(window: int, d: float, shape: int = 0) -> float:
    """sum_{(p,q) in W} exp(-(p^2+q^2)/d^2) over the disc (shape 0) or square (1) of radius `window`."""
    s = 0.0
    for p in range(-window, window + 1):
        for q in range(-window, window + 1):
            if shape == 0 and p * p + q * q > window * window:
                continue
            s += math.exp(-(p * p + q * q) / (d * d))
    return s


def repulsion_beta(window: int, d: float, shape: int = 0) -> float:
    """Reading Q24: beta * G_W = 0.2 * G_W(5x5 square, d = 5) of the Fig. 1 caption."""
    ref = 0.2 * window_weight_sum(2, 5.0, 1)
    return ref / window_weight_sum(window, d, shape)


def _rng(c: int, idx: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([BASE_SEED, c, idx])))


def _grid(M, N):
    ii, jj = np.meshgrid(np.arange(M, dtype=np.float64), np.arange(N, dtype=np.float64), indexing="ij")
    return ii, jj


def _paint_ellipse(img, ci, cj, a, b, theta, value):
    """Painter's-order fill of the rotated ellipse ((x'/a)^2 + (y'/b)^2 <= 1), pixel-centre test."""
    M, N = img.shape
    r = max(a, b)
    i0, i1 = max(0, int(math.floor(ci - r)) - 1), min(M, int(math.ceil(ci + r)) + 2)
    j0, j1 = max(0, int(math.floor(cj - r)) - 1), min(N, int(math.ceil(cj + r)) + 2)
    if i0 >= i1 or j0 >= j1:
        return
    ii, jj = np.meshgrid(np.arange(i0, i1, dtype=np.float64), np.arange(j0, j1, dtype=np.float64), indexing="ij")
    di, dj = ii - ci, jj - cj
    ct, st = math.cos(theta), math.sin(theta)
    x = ct * dj + st * di
    y = -st * dj + ct * di
    m = (x / a) ** 2 + (y / b) ** 2 <= 1.0
    img[i0:i1, j0:j1][m] = value


def _c1(rng):
    """configs[0]: 128^2, two unit disks r=20, centres 44 px apart (gap 4 px), noise 0.1."""
    M = N = 128
    ii, jj = _grid(M, N)
    img = np.zeros((M, N))
    for c in (41.5, 85.5):
        img[(ii - 63.5) ** 2 + (jj - c) ** 2 <= 400.0] = 1.0
    img += rng.normal(0.0, 0.1, size=(M, N))
    bj = -np.ones((M, N))
    bj[34:94, 12:116] = 1.0          # both disks' bounding box + 10 px margin
    return img, bj


def _c2(rng):
    """configs[1]: 512^2 annulus (r 60..120) + C-ring (r 60..90, 6 px opening) + 30x80 bar at 0.5."""
    M = N = 512
    ii, jj = _grid(M, N)
    img = np.zeros((M, N))
    r2a = (ii - 255.5) ** 2 + (jj - 150.0) ** 2
    img[(r2a >= 60.0 ** 2) & (r2a <= 120.0 ** 2)] = 1.0
    r2c = (ii - 255.5) ** 2 + (jj - 390.0) ** 2
    ring = (r2c >= 60.0 ** 2) & (r2c <= 90.0 ** 2)
    opening = (np.abs(ii - 255.5) < 3.0) & (jj > 390.0)
    img[ring & ~opening] = 1.0
    # occluding bar, axis-aligned, random orientation, centre uniform in the C-ring's bounding box
    h, w = (30, 80) if rng.random() < 0.5 else (80, 30)
    ci = rng.uniform(255.5 - 90.0, 255.5 + 90.0)
    cj = rng.uniform(390.0 - 90.0, 390.0 + 90.0)
    i0, i1 = int(round(ci - h / 2)), int(round(ci + h / 2))
    j0, j1 = int(round(cj - w / 2)), int(round(cj + w / 2))
    img[max(0, i0):min(M, i1), max(0, j0):min(N, j1)] = 0.5
    img += rng.normal(0.0, 0.2, size=(M, N))
    bj = np.where((ii - 255.5) ** 2 + (jj - 255.5) ** 2 <= 240.0 ** 2, 1.0, -1.0)
    return img, bj


def _ellipses(rng, M, N, n, amin, amax, cmin, cmax, noise):
    img = np.zeros((M, N))
    for _ in range(n):
        a, b = rng.uniform(amin, amax, size=2)
        theta = rng.uniform(0.0, math.pi)
        val = rng.uniform(0.6, 1.0)
        ci, cj = rng.uniform(cmin[0], cmax[0]), rng.uniform(cmin[1], cmax[1])
        _paint_ellipse(img, ci, cj, a, b, theta, val)
    img += rng.normal(0.0, noise, size=(M, N))
    return img


def _border_init(M, N, border):
    bj = -np.ones((M, N))
    bj[border:M - border, border:N - border] = 1.0
    return bj


def _c3_image(rng, M=1024, N=1024):
    """configs[2] (one image): 8..20 ellipses, semi-axes U(20,120), value U(0.6,1), noise 0.15."""
    n = int(rng.integers(8, 21))
    s = M / 1024.0
    img = _ellipses(rng, M, N, n, 20.0 * s, 120.0 * s, (64 * s, 64 * s), (M - 64 * s, N - 64 * s), 0.15)
    return img, _border_init(M, N, 16)


def _bezier(P, t):
    t = t[:, None]
    return ((1 - t) ** 3) * P[0] + 3 * ((1 - t) ** 2) * t * P[1] + 3 * (1 - t) * t * t * P[2] + (t ** 3) * P[3]


def _curve_samples(P):
    """Centreline samples at <= 0.25 px spacing."""
    coarse = _bezier(P, np.linspace(0.0, 1.0, 257))
    length = float(np.sum(np.hypot(*(np.diff(coarse, axis=0).T))))
    n = max(16, int(math.ceil(length / 0.25)) + 1)
    return _bezier(P, np.linspace(0.0, 1.0, n))


def _stamp_curve(img, pts, width):
    """Set pixels whose centre lies within width/2 of the sampled centreline."""
    M, N = img.shape
    r = width / 2.0
    k = int(math.ceil(r)) + 1
    base = np.floor(pts).astype(np.int64)
    offs = np.arange(-k, k + 1)
    for di in offs:
        for dj in offs:
            pi = base[:, 0] + di
            pj = base[:, 1] + dj
            d2 = (pi - pts[:, 0]) ** 2 + (pj - pts[:, 1]) ** 2
            ok = (d2 <= r * r) & (pi >= 0) & (pi < M) & (pj >= 0) & (pj < N)
            img[pi[ok], pj[ok]] = 1.0


def _c4(rng, M=4096, N=4096):
    """configs[3]: 40 thin curvilinear structures (20 pairs) of width 3..6 px coming within 2..8 px.

    Curve A of each pair is a cubic Bezier with control points U(128, M-128)^2.
    Curve B is A's offset curve along A's local normal at distance
    (w_A + w_B)/2 + gap(t), gap(t) = g0 + 1.5 sin(2 pi f t + p0) clipped to [2, 8],
    g0 ~ U(3.5, 6.5), so the pair's edge-to-edge gap stays within [2, 8] px.
    A pair is rejected if it comes within 2 px of an earlier pair.
    """
    from scipy.ndimage import gaussian_filter

    s = M / 4096.0
    img = np.zeros((M, N))
    occ = np.zeros((M, N))          # earlier pairs, dilated by 2 px + max half-width
    pairs = attempts = 0
    while pairs < 20 and attempts < 5000:
        attempts += 1
        PA = rng.uniform(128 * s, M - 128 * s, size=(4, 2))
        wA, wB = rng.uniform(3.0, 6.0, size=2)
        g0, f, p0 = rng.uniform(3.5, 6.5), rng.uniform(0.5, 3.0), rng.uniform(0, 2 * math.pi)
        sA = _curve_samples(PA)
        t = np.linspace(0.0, 1.0, len(sA))
        tan = np.gradient(sA, axis=0)
        tan /= np.linalg.norm(tan, axis=1, keepdims=True) + 1e-12
        nrm = np.stack([-tan[:, 1], tan[:, 0]], axis=1)
        gap = np.clip(g0 + 1.5 * np.sin(2 * math.pi * f * t + p0), 2.0, 8.0)
        sB = sA + nrm * ((wA + wB) / 2.0 + gap)[:, None]
        step = np.linalg.norm(np.diff(sB, axis=0), axis=1)
        if step.max() > 1.0:            # offset curve folds at high curvature: reject
            continue
        inb = lambda p: (p[:, 0] >= 0) & (p[:, 0] < M) & (p[:, 1] >= 0) & (p[:, 1] < N)
        if not (inb(sA).all() and inb(sB).all()):
            continue
        ia = np.floor(sA).astype(np.int64)
        ib = np.floor(sB).astype(np.int64)
        if occ[ia[:, 0], ia[:, 1]].any() or occ[ib[:, 0], ib[:, 1]].any():
            continue
        _stamp_curve(img, sA, wA)
        _stamp_curve(img, sB, wB)
        _stamp_curve(occ, sA, wA + 2 * (2.0 + 3.0) + 2)
        _stamp_curve(occ, sB, wB + 2 * (2.0 + 3.0) + 2)
        pairs += 1
    img += rng.normal(0.0, 0.1, size=(M, N))
    sm = gaussian_filter(img, 1.0, mode="nearest", truncate=3.0)
    bj = np.where(sm > 0.5, 1.0, -1.0)
    return img, bj


def _c5(rng, M=8192, N=8192):
    """configs[4]: 200 ellipses, semi-axes U(40,400), noise 0.15; phi0 +1 except a 32 px border."""
    s = M / 8192.0
    img = _ellipses(rng, M, N, 200, 40.0 * s, 400.0 * s, (256 * s, 256 * s), (M - 256 * s, N - 256 * s), 0.15)
    return img, _border_init(M, N, 32)


CONFIGS = {
    # name: (index in BASELINE.json configs, M, N, batch, K, window radius R)
    "c1": dict(index=0, M=128, N=128, batch=1, K=300, window=3),
    "c2": dict(index=1, M=512, N=512, batch=1, K=500, window=4),
    "c3": dict(index=2, M=1024, N=1024, batch=64, K=1000, window=4),
    "c4": dict(index=3, M=4096, N=4096, batch=1, K=500, window=6),
    "c5": dict(index=4, M=8192, N=8192, batch=1, K=300, window=5),
}


def make_config(name: str, images=None, size=None) -> dict:
    """Generate config `name` ("c1".."c5").

    images : optional iterable of image indices (C3 only; default all 64).
    size   : optional (M, N) override for the scalable generators (C3, C4, C5)
             so tests can run the same recipe at a size the oracle finishes.
    Returns dict(name, image f32[B,M,N], phi0 f32[B,M,N] (paper convention, phi<0 inside),
    params, K).
    """
    cfg = dict(CONFIGS[name])
    c = cfg["index"] + 1
    if name == "c3":
        idx = list(range(cfg["batch"])) if images is None else list(images)
        M, N = size if size else (cfg["M"], cfg["N"])
        ims, phis = [], []
        for k in idx:
            im, bj = _c3_image(_rng(c, k), M, N)
            ims.append(im)
            phis.append(-bj)
        image, phi0 = np.stack(ims), np.stack(phis)
    else:
        rng = _rng(c)
        if name == "c1":
            im, bj = _c1(rng)
        elif name == "c2":
            im, bj = _c2(rng)
        elif name == "c4":
            im, bj = _c4(rng, *(size or (cfg["M"], cfg["N"])))
        else:
            im, bj = _c5(rng, *(size or (cfg["M"], cfg["N"])))
        image, phi0 = im[None], (-bj)[None]
    return dict(name=name, image=np.ascontiguousarray(image, dtype=np.float32),
                phi0=np.ascontiguousarray(phi0, dtype=np.float32),
                params=paper_params(cfg["window"]), K=cfg["K"])


def random_state(M, N, batch=1, seed=0, band=True):
    """Random solver state (phi, w1, w2, b1, b2, g, image) for teacher-forced kernel parity tests.

    phi is smooth-ish with values spread over [-1.5, 1.5] so the narrow band
    (|phi| <= l + eps) is well populated; w, b are O(1); g in (0, 1].
    """
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([BASE_SEED, 99, seed, M, N, batch])))
    ii, jj = _grid(M, N)
    out = {k: [] for k in ("phi", "w1", "w2", "b1", "b2", "g", "image")}
    for _ in range(batch):
        k1, k2 = rng.uniform(0.02, 0.2, size=2)
        ph = 1.2 * np.sin(k1 * ii + rng.uniform(0, 6.3)) * np.cos(k2 * jj + rng.uniform(0, 6.3))
        ph += 0.3 * rng.standard_normal((M, N))
        if not band:
            ph = np.clip(ph * 3, -1, 1)
        out["phi"].append(ph)
        out["w1"].append(rng.uniform(-1, 1, (M, N)))
        out["w2"].append(rng.uniform(-1, 1, (M, N)))
        out["b1"].append(0.3 * rng.standard_normal((M, N)))
        out["b2"].append(0.3 * rng.standard_normal((M, N)))
        out["g"].append(rng.uniform(0.05, 1.0, (M, N)))
        out["image"].append(rng.uniform(0, 1, (M, N)))
    return {k: np.ascontiguousarray(np.stack(v), dtype=np.float32) for k, v in out.items()}
