"""Full-size checks in the launch configuration bench.py times (BASELINE configs at their real
sizes): properties that hold at any size (the fp64 residual of the GPU's phi solve) and oracle
comparisons of the RHS and w/b kernels on crops.  The RHS / w/b output at a pixel depends only on
its (window + 1)-neighbourhood, so the oracle run on a crop with a margin of window + 2 pixels (or
the true image border) reproduces the interior of the crop exactly."""
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
    return srsb


def _periodic_residual(phi, F, tau, mu):
    lap = (np.roll(phi, 1, 0) + np.roll(phi, -1, 0) + np.roll(phi, 1, 1) + np.roll(phi, -1, 1) - 4 * phi)
    return np.linalg.norm(phi - tau * mu * lap - F) / np.linalg.norm(F)


def _state(M, N, B, seed):
    """Random band-populated state generated on the GPU (torch.Generator, seeded): inputs only."""
    gen = torch.Generator(device="cuda").manual_seed(seed)
    u = lambda *s: torch.rand(*s, generator=gen, device="cuda")
    phi = (2.4 * u(B, M, N) - 1.2).contiguous()
    w = (2 * u(B, 2, M, N) - 1).contiguous()
    b = (0.6 * u(B, 2, M, N) - 0.3).contiguous()
    g = (0.05 + 0.95 * u(B, M, N)).contiguous()
    return phi, w, b, g


CASES = [("c3", 1024, 1024, 64, 4), ("c4", 4096, 4096, 1, 6), ("c5", 8192, 8192, 1, 5)]


@pytest.mark.parametrize("name,M,N,B,R", CASES)
def test_fullsize_solve_residual(S, name, M, N, B, R):
    from synth import paper_params
    p = paper_params(R)
    with S.Solver(M, N, B, window=R, **{k: p[k] for k in KEYS}) as sv:
        gen = torch.Generator(device="cuda").manual_seed(7)
        F = torch.randn(B, M, N, generator=gen, device="cuda")
        phi = sv.debug_solve(F)
        torch.cuda.synchronize()
        for b in sorted({0, B - 1}):
            res = _periodic_residual(phi[b].double().cpu().numpy(), F[b].double().cpu().numpy(), p["tau"], p["mu"])
            assert res < 2e-6, res


def _crops(M, N, R):
    m = R + 2
    c = 48
    return [(0, 0), (0, N - c), (M - c, 0), (M - c, N - c), (M // 2 - 17, N // 3 + 5), (m + 3, N // 2)], c, m


@pytest.mark.parametrize("name,M,N,B,R", CASES)
def test_fullsize_rhs_and_wb_on_crops(S, orc, name, M, N, B, R):
    from synth import paper_params
    p = paper_params(R)
    phi, w, b, g = _state(M, N, B, seed=11)
    with S.Solver(M, N, B, window=R, **{k: p[k] for k in KEYS}) as sv:
        sv.set_state(phi, w, b, g)
        D = sv.debug_rhs().cpu().numpy()
        sv.debug_wb()
        st = sv.get_state()
        w_new, b_new = st["w"].cpu().numpy(), st["b"].cpu().numpy()
    phi_h, w_h, b_h, g_h = (t.cpu().numpy() for t in (phi, w, b, g))   # float32; crops go to float64
    crops, c, m = _crops(M, N, R)
    for img in sorted({0, B - 1}):
        for (i0, j0) in crops:
            # crop with margin m, clipped to the image (true borders need no margin)
            a0, a1 = max(i0 - m, 0), min(i0 + c + m, M)
            b0, b1 = max(j0 - m, 0), min(j0 + c + m, N)
            sl = (slice(a0, a1), slice(b0, b1))
            f64 = lambda x: np.ascontiguousarray(x[sl], dtype=np.float64)
            psi = f64(phi_h[img])
            args = (psi, f64(w_h[img, 0]), f64(w_h[img, 1]), f64(b_h[img, 0]), f64(b_h[img, 1]), f64(g_h[img]))
            F = orc.rhs(p, *args)
            inner = (slice(i0 - a0, i0 - a0 + c), slice(j0 - b0, j0 - b0 + c))
            # increment form D = F - psi + tau mu Delta_per psi, Delta_per the periodic 5-point
            # Laplacian of the WHOLE image: rows / columns of the crop block taken modulo M, N
            ri = np.arange(i0 - 1, i0 + c + 1) % M
            cj = np.arange(j0 - 1, j0 + c + 1) % N
            blk = phi_h[img][np.ix_(ri, cj)].astype(np.float64)
            lap = blk[:-2, 1:-1] + blk[2:, 1:-1] + blk[1:-1, :-2] + blk[1:-1, 2:] - 4 * blk[1:-1, 1:-1]
            Dref = F[inner] - psi[inner] + p["tau"] * p["mu"] * lap
            Dg = D[img, i0:i0 + c, j0:j0 + c]
            assert np.max(np.abs(Dg - Dref) / (1 + np.abs(F[inner]))) < 2e-5, (name, img, i0, j0)
            r1, r2, rb1, rb2 = orc.wb(p, *args)
            for got, ref in ((w_new[img, 0], r1), (w_new[img, 1], r2), (b_new[img, 0], rb1), (b_new[img, 1], rb2)):
                assert np.max(np.abs(got[i0:i0 + c, j0:j0 + c] - ref[inner])) < 2e-5, (name, img, i0, j0)


def test_fullsize_aos_solve_sampled(S, orc):
    """NEXT-4 at the bench launch configuration (C3: 64 x 1024^2, --phi-solver aos): the AOS solve
    of random fields against the oracle's, on the first and last image."""
    from synth import paper_params
    p = paper_params(4)
    B, M, N = 64, 1024, 1024
    with S.Solver(M, N, B, window=4, phi_solver=1, **{k: p[k] for k in KEYS}) as sv:
        gen = torch.Generator(device="cuda").manual_seed(11)
        F = torch.randn(B, M, N, generator=gen, device="cuda")
        phi = sv.debug_solve(F)
        torch.cuda.synchronize()
        for b in (0, B - 1):
            ref = orc.solve_aos(F[b].double().cpu().numpy(), p["tau"], p["mu"])
            assert np.max(np.abs(phi[b].double().cpu().numpy() - ref)) <= 2e-6 * float(F[b].abs().max())


def test_fullsize_3d_solve_residual(S):
    """NEXT-3 at the bench size (one 128^3 volume): fp64 residual of the GPU's 3-D solve with the
    periodic 7-point operator (a property that holds at any size)."""
    from synth import paper_params3
    p = paper_params3(3)
    D = M = N = 128
    with S.Solver3(D, M, N, window=3, **{k: p[k] for k in KEYS}) as sv:
        gen = torch.Generator(device="cuda").manual_seed(13)
        F = torch.randn(D, M, N, generator=gen, device="cuda")
        phi = sv.debug_solve(F).double().cpu().numpy()
    Fd = F.double().cpu().numpy()
    lap = sum(np.roll(phi, s, a) for a in range(3) for s in (1, -1)) - 6 * phi
    res = np.linalg.norm(phi - p["tau"] * p["mu"] * lap - Fd) / np.linalg.norm(Fd)
    assert res < 2e-6, res
