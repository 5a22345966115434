"""Checkpoint / resume through the C ABI (SURVEY §8(b) get_state / set_state + the iteration
counter): K1 iterations, save, restore into a fresh context, K2 more == K1 + K2 uninterrupted,
bitwise (same kernels, same order)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

KEYS = ("gamma", "alpha", "beta", "mu", "epsilon", "l", "d", "window_shape", "tau", "S", "rho", "sigma", "s",
        "phi_clip", "w_proj", "w_mode", "w_iters")


def test_checkpoint_resume_bitwise():
    from paper_2003_12693_b200 import Solver
    from synth import make_config
    c = make_config("c2")
    p = c["params"]
    B, M, N = c["image"].shape
    img = torch.from_numpy(c["image"]).cuda()
    phi0 = torch.from_numpy(c["phi0"]).cuda()
    with Solver(M, N, B, window=p["window"], **{k: p[k] for k in KEYS}) as a:
        a.set_image(img, phi0)
        a.iterate(7)
        ref = a.get_phi().cpu().numpy()
    with Solver(M, N, B, window=p["window"], **{k: p[k] for k in KEYS}) as a:
        a.set_image(img, phi0)
        a.iterate(3)
        st = a.get_state()
        k = a.iteration
    assert k == 3
    with Solver(M, N, B, window=p["window"], **{k: p[k] for k in KEYS}) as b:
        b.set_state(st["phi"], st["w"], st["b"], st["g"])
        b.iteration = k
        b.iterate(4)
        assert b.iteration == 7
        out = b.get_phi().cpu().numpy()
    assert np.array_equal(out, ref)
