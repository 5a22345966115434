"""GPU parity of the 3-D extension (NEXT-3, reading Q26) through the C ABI (sr_sb3_*), against the
3-D float64 oracle pinned in tests/test_oracle_3d.py."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

KEYS = ("gamma", "alpha", "beta", "mu", "epsilon", "l", "d", "window_shape", "tau", "S", "rho", "sigma", "s",
        "phi_clip", "w_proj", "w_mode", "w_iters")


@pytest.fixture(scope="module")
def S():
    from paper_2003_12693_b200 import build
    build.build()
    from paper_2003_12693_b200 import srsb
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return srsb


def _p(window, **over):
    from synth import paper_params3
    return paper_params3(window, **over)


def _solver(S, shape, p):
    D, M, N = shape
    return S.Solver3(D, M, N, window=p["window"], **{k: p[k] for k in KEYS})


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _np(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy().astype(np.float64)


def _rand(shape, seed, lo=-1.0, hi=1.0):
    return np.random.default_rng(seed).uniform(lo, hi, shape)


@pytest.mark.parametrize("shape", [(1, 8, 8), (2, 8, 16), (8, 16, 32), (16, 16, 16), (32, 64, 32), (64, 128, 64),
                                   (128, 128, 128), (16, 8, 256), (16, 32, 16), (64, 512, 32), (256, 256, 64)])
@pytest.mark.parametrize("path", ["default", "plane"])
def test_solve3_parity(S, orc, shape, path, monkeypatch):
    """path: the default solve (FFT along j and i + cyclic tridiagonal solve along z where D >= 16 and M >= 32,
    any size; else one D x M spectrum plane in shared memory) or the plane solve forced (needs D (M + 1) <= 25600:
    the last two shapes exist only on the default path)."""
    D, M, N = shape
    if path == "plane":
        if D * (M + 1) > 25600:
            pytest.skip("beyond the plane solve's shared-memory limit")
        monkeypatch.setenv("SRSB_VOL_SOLVE", "plane")
    p = _p(2)
    F = _rand(shape, sum(shape)).astype(np.float32)
    with _solver(S, shape, p) as sv:
        out = _np(sv.debug_solve(_cuda(F)))
    ref = orc.solve3(F, p["tau"], p["mu"])
    assert np.max(np.abs(out - ref)) <= 2e-6 * np.max(np.abs(F))


@pytest.mark.parametrize("D,M,N", [(8, 16, 32), (32, 32, 32)])
def test_solve3_cos_modes(S, D, M, N):
    """A single cosine mode (k3, k1, k2), including the packed k2 = 0 and N/2 columns, is scaled by
    1 / symbol (Eq. 32 in 3-D); the second shape runs the lines solve (unpacked k2 = 0 / N/2 planes)."""
    p = _p(2)
    tm = p["tau"] * p["mu"]
    z, i, j = np.meshgrid(np.arange(D), np.arange(M), np.arange(N), indexing="ij")
    for k3, k1, k2 in [(0, 0, 0), (1, 0, 0), (0, 3, 0), (2, 5, 0), (3, 1, N // 2), (D // 2, M // 2, N // 2),
                       (1, 2, 7), (D - 1, M - 1, 1)]:
        F = np.cos(2 * np.pi * (k3 * z / D + k1 * i / M + k2 * j / N)).astype(np.float32)
        sig = 1 + tm * (6 - 2 * np.cos(2 * np.pi * k3 / D) - 2 * np.cos(2 * np.pi * k1 / M) - 2 * np.cos(2 * np.pi * k2 / N))
        with _solver(S, (D, M, N), p) as sv:
            out = _np(sv.debug_solve(_cuda(F)))
        assert np.max(np.abs(out - F / sig)) < 2e-6, (k3, k1, k2)


def test_edge3_and_init_parity(S, orc):
    shape = (8, 16, 32)
    p = _p(2)
    vol = _rand(shape, 3, 0, 1)
    phi0 = np.where(_rand(shape, 4) > 0, 1.0, -1.0)
    with _solver(S, shape, p) as sv:
        sv.set_image(_cuda(vol), _cuda(phi0))
        st = sv.get_state()
        g, w, b, phi = _np(st["g"]), _np(st["w"]), _np(st["b"]), _np(st["phi"])
    assert np.max(np.abs(g - orc.edge3(vol, p["sigma"], p["rho"], p["s"]))) < 2e-6
    for c, ref in enumerate(orc.grad3(phi0)):
        assert np.array_equal(w[c], ref)
    assert not b.any() and np.array_equal(phi, phi0)


def _state(shape, seed):
    from synth import random_state
    rng = np.random.default_rng(seed)
    phi = np.clip(1.2 * np.sin(rng.uniform(0.1, 0.4) * np.arange(shape[0]))[:, None, None]
                  * np.cos(rng.uniform(0.05, 0.3) * np.arange(shape[1]))[None, :, None]
                  + 0.3 * rng.standard_normal(shape), -1.5, 1.5)
    w = rng.uniform(-1, 1, (3,) + shape)
    b = 0.3 * rng.standard_normal((3,) + shape)
    g = rng.uniform(0.1, 1.0, shape)
    del random_state
    return phi, w, b, g


def _periodic_lap3(phi):
    return sum(np.roll(phi, s, a) for a in range(3) for s in (1, -1)) - 6 * phi


@pytest.mark.parametrize("shape,window,wshape,eps,l", [((8, 16, 32), 1, 0, 0.5, 0.5), ((8, 16, 64), 2, 0, 0.5, 0.5),
                                                       ((16, 16, 32), 3, 0, 0.5, 0.5), ((8, 8, 32), 4, 0, 0.5, 0.5),
                                                       ((8, 16, 32), 2, 1, 0.5, 0.5), ((8, 16, 32), 2, 0, 0.7, 0.3),
                                                       ((4, 8, 8), 0, 0, 0.5, 0.5)])
def test_rhs3_parity(S, orc, shape, window, wshape, eps, l):
    p = _p(window, window_shape=wshape, epsilon=eps, l=l)
    phi, w, b, g = _state(shape, window + 10 * wshape)
    with _solver(S, shape, p) as sv:
        sv.set_state(_cuda(phi), _cuda(w), _cuda(b), _cuda(g))
        Dg = _np(sv.debug_rhs())
    F = orc.rhs3(p, phi, tuple(w), tuple(b), g)
    Dref = F - phi + p["tau"] * p["mu"] * _periodic_lap3(phi)
    assert np.max(np.abs(Dg - Dref) / (1 + np.abs(F))) < 2e-5


@pytest.mark.parametrize("window,mode,iters", [(2, 0, 1), (3, 0, 1), (2, 1, 2)])
def test_wb3_parity(S, orc, window, mode, iters):
    shape = (8, 16, 32)
    p = _p(window, w_mode=mode, w_iters=iters)
    phi, w, b, g = _state(shape, 40 + window)
    phi = np.clip(phi, -1, 1)
    with _solver(S, shape, p) as sv:
        sv.set_state(_cuda(phi), _cuda(w), _cuda(b), _cuda(g))
        sv.iterate(1)                    # one iteration: S sweeps then the w/b update from the new phi
        st = sv.get_state()
        phig, wg, bg = _np(st["phi"]), _np(st["w"]), _np(st["b"])
    ref = {"phi": phi, "w": tuple(w), "b": tuple(b)}
    orc.iterate3(p, ref, g, 1)
    assert np.max(np.abs(phig - ref["phi"])) < 2e-5
    for c in range(3):
        assert np.max(np.abs(wg[c] - ref["w"][c])) < 1e-4
        assert np.max(np.abs(bg[c] - ref["b"][c])) < 1e-4


def test_trajectory3(S, orc):
    """Algorithm 1 in 3-D, free running for 10 iterations on the synthetic volume recipe."""
    from synth import make_volume
    v = make_volume((16, 32, 32), n=5, window=2, seed=3, border=2)
    p = v["params"]
    with _solver(S, v["volume"].shape, p) as sv:
        sv.set_image(_cuda(v["volume"]), _cuda(v["phi0"]))
        errs = []
        st = None
        for k in range(10):
            sv.iterate(1)
            phi = _np(sv.get_phi())
            if st is None:
                g = orc.edge3(v["volume"], p["sigma"], p["rho"], p["s"])
                st = orc.init3(v["phi0"])
            orc.iterate3(p, st, g, 1)
            errs.append(float(np.max(np.abs(phi - st["phi"]))))
        sv.sync()
    assert max(errs) <= 1e-4, errs


def test_graph_and_direct_agree(S):
    from synth import make_volume
    v = make_volume((8, 16, 32), n=3, window=2, seed=5, border=2)
    p = v["params"]
    outs = []
    for chunks in ([6], [1, 1, 1, 1, 1, 1]):
        with _solver(S, v["volume"].shape, p) as sv:
            sv.set_image(_cuda(v["volume"]), _cuda(v["phi0"]))
            for k in chunks:
                sv.iterate(k)
            outs.append(_np(sv.get_phi()))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("size,window", [((32, 64, 64), 3), ((64, 64, 64), 4), ((16, 32, 64), 2)])
def test_band_skip3_is_exact(S, monkeypatch, size, window):
    """The 3-D narrow-band skip of the ball sums (sr_vol.cuh vol_v) drops only terms multiplied by an
    exact zero: free-running states with and without it are bitwise equal."""
    from synth import make_volume
    v = make_volume(size, n=6, window=window, seed=11, border=3)
    p = v["params"]

    def run():
        with _solver(S, v["volume"].shape, p) as sv:
            sv.set_image(_cuda(v["volume"]), _cuda(v["phi0"]))
            sv.iterate(6)
            st = sv.get_state()
            out = {k: t.cpu().numpy() for k, t in st.items()}
            sv.sync()
        return out
    a = run()
    monkeypatch.setenv("SRSB_BAND_SKIP", "0")
    b = run()
    for k in ("phi", "w", "b"):
        assert np.array_equal(a[k], b[k]), k
