"""The fused RHS + row R2C cluster kernel (k_rhs_r2c) through the C ABI.

It runs the same arithmetic in the same order as k_rhs_tma -> k_rows_r2c (the D tile stays in
shared memory, the row transforms gather it through distributed shared memory), so whole-image
trajectories must be BITWISE equal with and without it (SRSB_FUSE=0).  The unfused path is the one
tests/test_gpu_parity.py holds to the float64 oracle (the fused kernel is opt-in, SRSB_FUSE=1: it
measured slower); here: bitwise identity on
shapes that span the cluster sizes 2..16 (N = 128..1024), ragged bands (M < 32), batches, every
window shape, l != eps, the fixed-point w mode, and the monitor.
"""
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
    assert torch.cuda.is_available()
    return srsb


def _run(S, M, N, B, window, K, seed, monitor=False, **over):
    from synth import paper_params, random_state
    p = paper_params(window)
    p.update(over)
    rs = random_state(M, N, batch=B, seed=seed)
    with S.Solver(M, N, B, window=window, **{k: p[k] for k in KEYS}) as sv:
        fused = sv.launches_per_iteration == 3 * p["S"] + (p["w_iters"] if p["w_mode"] == 1 else 1)
        img = torch.from_numpy(rs["image"]).cuda()
        phi0 = torch.from_numpy(np.clip(rs["phi"], -1, 1).astype(np.float32)).cuda()
        sv.set_image(img, phi0)
        if monitor:
            sv.set_monitor(True)
        sv.iterate(K)
        st = sv.get_state()
        mon = sv.monitor() if monitor else None
        out = {k: v.cpu().numpy() for k, v in st.items()}
        sv.sync()
    return fused, out, mon


@pytest.mark.parametrize("M,N,B,window,over", [
    (128, 128, 1, 3, {}),
    (256, 256, 2, 4, {}),
    (512, 512, 1, 4, {}),
    (1024, 1024, 2, 4, {}),
    (64, 1024, 3, 5, {}),
    (16, 512, 2, 2, {}),
    (8, 128, 1, 1, {}),
    (256, 128, 1, 6, {"window_shape": 1}),
    (128, 256, 2, 3, {"epsilon": 0.5, "l": 1.0}),
    (256, 512, 1, 4, {"w_mode": 1, "w_iters": 2}),
    (128, 1024, 1, 8, {}),
    (256, 256, 1, 0, {}),
])
def test_fused_bitwise_equals_unfused(S, monkeypatch, M, N, B, window, over):
    K = 5
    # both sides on the transposed spectrum with the separate column / c2r passes (the fused kernel writes that
    # layout; the row-major spectrum and the one-kernel cluster solve are other rounding orders)
    monkeypatch.setenv("SRSB_SPEC_RM", "0")
    monkeypatch.setenv("SRSB_SOLVE_CL", "0")
    monkeypatch.setenv("SRSB_FUSE", "1")
    fused, a, _ = _run(S, M, N, B, window, K, seed=M + N + window, **over)
    assert fused, "the fused kernel was not selected for this shape"
    monkeypatch.setenv("SRSB_FUSE", "0")
    unfused, b, _ = _run(S, M, N, B, window, K, seed=M + N + window, **over)
    assert not unfused
    for k in ("phi", "w", "b"):
        assert np.array_equal(a[k], b[k]), k


def test_fused_monitor_and_profile(S, monkeypatch):
    """Monitor sums (energies, per-sweep changes) agree with the unfused run to fp64 atomic order; the
    profile reports the fused class (rhs_r2c) with S launches per iteration and no rhs / rows_r2c."""
    monkeypatch.setenv("SRSB_FUSE", "1")
    _, a, ma = _run(S, 256, 256, 2, 4, 3, seed=5, monitor=True)
    monkeypatch.setenv("SRSB_FUSE", "0")
    _, b, mb = _run(S, 256, 256, 2, 4, 3, seed=5, monitor=True)
    assert np.array_equal(a["phi"], b["phi"])
    for x, y in zip(ma, mb):
        for key in ("E_g", "E_a", "E_r", "E_pen"):
            np.testing.assert_allclose(x[key], y[key], rtol=1e-9, atol=1e-9)
        np.testing.assert_allclose(x["sweep_change"], y["sweep_change"], rtol=1e-9, atol=1e-12)
    monkeypatch.setenv("SRSB_FUSE", "1")
    from synth import paper_params
    p = paper_params(4)
    with S.Solver(256, 256, 1, window=4, **{k: p[k] for k in KEYS}) as sv:
        sv.set_image(torch.zeros(1, 256, 256, device="cuda"), -torch.ones(1, 256, 256, device="cuda"))
        prof = sv.profile(2)
        sv.sync()
    assert prof["rhs_r2c"][1] == 2 * p["S"]
    assert "rhs" not in prof and "rows_r2c" not in prof
    assert prof["cols_solve"][1] == 2 * p["S"] and prof["rows_c2r"][1] == 2 * p["S"]


def test_fused_not_used_where_it_does_not_apply(S, monkeypatch):
    """N = 2048 (cluster would exceed 16 CTAs) and the AOS solver keep the unfused path."""
    monkeypatch.setenv("SRSB_FUSE", "1")
    from synth import paper_params
    p = paper_params(4)
    with S.Solver(64, 2048, 1, window=4, **{k: p[k] for k in KEYS}) as sv:
        assert sv.launches_per_iteration == 4 * p["S"] + 1
    with S.Solver(128, 128, 1, window=4, phi_solver=1, **{k: p[k] for k in KEYS}) as sv:
        assert sv.launches_per_iteration == 3 * p["S"] + 1
