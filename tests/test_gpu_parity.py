"""GPU parity: every kernel of the hot path, through the C ABI, against the float64 oracle on the
same seeded inputs (DESIGN.md §6 for the tolerances and where they come from).

Kernel-level (teacher-forced) checks compare each step on random states that span several
tiles and a ragged tail; the trajectory checks run Algorithm 1 free for 10 iterations on the
BASELINE configs (tolerance 1e-4 from north_star) and to completion on C1 (masks).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    from paper_2003_12693_b200 import build
    build.build()
    from paper_2003_12693_b200 import srsb
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return srsb


def _params(window, **over):
    from synth import paper_params
    p = paper_params(window)
    p.update(over)
    return p


def _solver(S, M, N, batch, p):
    keys = ("gamma", "alpha", "beta", "mu", "epsilon", "l", "d", "window_shape", "tau", "S", "rho", "sigma",
            "s", "phi_clip", "w_proj", "w_mode", "w_iters")
    return S.Solver(M, N, batch, window=p["window"], **{k: p[k] for k in keys})


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def _np(t):
    torch.cuda.synchronize()
    return t.detach().cpu().numpy().astype(np.float64)


def _periodic_residual(phi, F, tau, mu):
    lap = (np.roll(phi, 1, 0) + np.roll(phi, -1, 0) + np.roll(phi, 1, 1) + np.roll(phi, -1, 1) - 4 * phi)
    return np.linalg.norm(phi - tau * mu * lap - F) / np.linalg.norm(F)


def _cols_env(monkeypatch, cols):
    """Variants of the phi solve (knobs read at context creation): 'cl' = the one-kernel cluster solve forced
    wherever it applies (M <= 512, 128 <= N <= 512; by default only up to 128 x 128), else the defaults; 'rm' = cyclic
    tridiagonal column pass on the row-major spectrum (N >= 64, M >= 16, short carries); 'tri' = the same on
    the transposed spectrum (contiguous columns); 'fft' = FFT -> divide by the symbol -> inverse FFT."""
    monkeypatch.setenv("SRSB_COLS_TRI", "0" if cols == "fft" else "1")
    if cols == "cl":
        monkeypatch.setenv("SRSB_SOLVE_CL", "1")
        monkeypatch.delenv("SRSB_SPEC_RM", raising=False)
    else:
        monkeypatch.setenv("SRSB_SOLVE_CL", "0")
        monkeypatch.setenv("SRSB_SPEC_RM", "1" if cols == "rm" else "0")


# ----------------------------------------------------------------------------- FFT solve, Eq. (33)
@pytest.mark.parametrize("M,N,batch", [(8, 8, 1), (16, 64, 2), (64, 16, 1), (128, 128, 1), (32, 512, 1),
                                       (512, 32, 1), (256, 256, 3), (1024, 1024, 2), (2048, 256, 1),
                                       (256, 4096, 1), (8192, 16, 1), (16, 8192, 1)])
@pytest.mark.parametrize("cols", ["cl", "rm", "tri", "fft"])
def test_solve_parity(S, orc, M, N, batch, cols, monkeypatch):
    _cols_env(monkeypatch, cols)
    p = _params(3)
    rng = np.random.default_rng(M * 7 + N)
    F = rng.standard_normal((batch, M, N)).astype(np.float32)
    with _solver(S, M, N, batch, p) as sv:
        out = _np(sv.debug_solve(_cuda(F)))
    for b in range(batch):
        ref = orc.solve(F[b], p["tau"], p["mu"])
        err = np.max(np.abs(out[b] - ref))
        assert err <= 1e-5 * np.max(np.abs(F[b])), (b, err)
        assert _periodic_residual(out[b], F[b].astype(np.float64), p["tau"], p["mu"]) < 2e-6


@pytest.mark.parametrize("M,N,tau,mu", [(16, 64, 0.05, 8.0), (16, 16, 5.0, 8.0), (64, 64, 5.0, 20.0),
                                        (1024, 256, 1.0, 8.0), (1024, 1024, 30.0, 8.0), (4096, 64, 0.5, 8.0),
                                        (256, 256, 0.0, 8.0), (128, 128, 1e-4, 1.0), (512, 128, 0.25, 8.0),
                                        (64, 128, 0.3, 8.0), (128, 256, 5.0, 20.0), (512, 512, 30.0, 8.0),
                                        (256, 128, 0.05, 8.0), (32, 512, 0.05, 8.0)])
@pytest.mark.parametrize("cols", ["cl", "rm", "tri"])
def test_solve_tridiagonal_column_pass_any_stiffness(S, orc, M, N, tau, mu, cols, monkeypatch):
    """sr_tri.cuh: the carry sum of the chunked recurrences must hold from r = 0 (tau = 0) to r -> 1
    (tau mu = 240: r = 0.94, carries that wrap around the whole column; the row-major kernel takes up to
    4 carry terms and hands stiffer cases to the transposed one)."""
    _cols_env(monkeypatch, cols)
    p = _params(3, tau=tau, mu=mu)
    rng = np.random.default_rng(M * 11 + N)
    F = rng.standard_normal((2, M, N)).astype(np.float32)
    F[1] = 0.0
    F[1, M // 3, N // 5] = 1.0          # an impulse: the Green's function itself, wrap included
    with _solver(S, M, N, 2, p) as sv:
        out = _np(sv.debug_solve(_cuda(F)))
    for b in range(2):
        ref = orc.solve(F[b], tau, mu)
        assert np.max(np.abs(out[b] - ref)) <= 1e-5 * np.max(np.abs(F[b])), b
        # fp32 rounding of phi seen through A: up to (1 + 8 tau mu) eps |phi|
        assert _periodic_residual(out[b], F[b].astype(np.float64), tau, mu) < 2e-6 * (1 + 8 * tau * mu)


@pytest.mark.parametrize("cols", ["cl", "rm", "tri", "fft"])
def test_solve_closed_forms(S, cols, monkeypatch):
    """Constant -> same constant; a single cos mode (k1, k2), including the packed k2 = 0 and
    k2 = N/2 columns, -> scaled by 1/symbol (Eq. 32)."""
    _cols_env(monkeypatch, cols)
    M, N = 64, 128
    tau, mu = _params(3)["tau"], _params(3)["mu"]
    ii, jj = np.meshgrid(np.arange(M), np.arange(N), indexing="ij")
    modes = [(0, 0), (1, 0), (0, N // 2), (M // 2, N // 2), (5, 0), (7, N // 2), (3, 17), (M - 1, 1)]
    F = np.stack([np.cos(2 * np.pi * (k1 * ii / M + k2 * jj / N)) for k1, k2 in modes]).astype(np.float32)
    with _solver(S, M, N, len(modes), _params(3)) as sv:
        out = _np(sv.debug_solve(_cuda(F)))
    for b, (k1, k2) in enumerate(modes):
        sig = 1 + tau * mu * (4 - 2 * np.cos(2 * np.pi * k1 / M) - 2 * np.cos(2 * np.pi * k2 / N))
        assert np.max(np.abs(out[b] - F[b] / sig)) < 2e-6, (k1, k2)


# ----------------------------------------------------------------------------- edge indicator, init
@pytest.mark.parametrize("M,N", [(128, 128), (8, 64), (256, 512)])
def test_edge_and_init_parity(S, orc, M, N):
    from synth import random_state
    st = random_state(M, N, batch=2, seed=3)
    p = _params(4)
    with _solver(S, M, N, 2, p) as sv:
        sv.set_image(_cuda(st["image"]), _cuda(st["phi"]))
        s = sv.get_state()
        g, w, b, phi = _np(s["g"]), _np(s["w"]), _np(s["b"]), _np(s["phi"])
    for k in range(2):
        gref = orc.edge(st["image"][k], p["sigma"], p["rho"], p["s"])
        assert np.max(np.abs(g[k] - gref)) < 2e-6
        g1, g2 = orc.grad(st["phi"][k])
        assert np.max(np.abs(w[k, 0] - g1)) < 1e-6 and np.max(np.abs(w[k, 1] - g2)) < 1e-6
        assert not b[k].any()
        assert np.array_equal(phi[k], st["phi"][k])


# ----------------------------------------------------------------------------- RHS, Eq. (37)
@pytest.mark.parametrize("M,N,window,shape,eps,l", [(64, 64, 3, 0, 0.5, 0.5), (128, 256, 4, 0, 0.5, 0.5),
                                                     (128, 512, 6, 0, 0.5, 0.5), (8, 16, 4, 0, 0.5, 0.5),
                                                     (16, 1024, 5, 1, 0.5, 0.5), (256, 128, 8, 0, 0.5, 0.5),
                                                     (32, 32, 0, 0, 0.5, 0.5), (128, 128, 2, 1, 0.5, 0.5),
                                                     (128, 256, 4, 0, 0.7, 0.3), (64, 128, 3, 1, 1.0, 1.0)])
def test_rhs_parity(S, orc, M, N, window, shape, eps, l):
    from synth import random_state
    st = random_state(M, N, batch=2, seed=window)
    p = _params(window, window_shape=shape, d=max(window, 1) * 0.9, epsilon=eps, l=l)
    with _solver(S, M, N, 2, p) as sv:
        w = np.stack([st["w1"], st["w2"]], 1)
        b = np.stack([st["b1"], st["b2"]], 1)
        sv.set_state(_cuda(st["phi"]), _cuda(w), _cuda(b), _cuda(st["g"]))
        F = _np(sv.debug_rhs())
    for k in range(2):
        ref = orc.rhs(p, st["phi"][k], st["w1"][k], st["w2"][k], st["b1"][k], st["b2"][k], st["g"][k])
        # the library returns the increment form D = F - (1 - tau mu Delta_per) psi
        psi = st["phi"][k].astype(np.float64)
        lap = np.roll(psi, 1, 0) + np.roll(psi, -1, 0) + np.roll(psi, 1, 1) + np.roll(psi, -1, 1) - 4 * psi
        Dref = ref - psi + p["tau"] * p["mu"] * lap
        err = np.abs(F[k] - Dref) / (1 + np.abs(ref))
        assert err.max() < 2e-5, (k, err.max(), np.unravel_index(err.argmax(), err.shape))


# ----------------------------------------------------------------------------- w/b update, Eq. (41),(42),(40),(23)
@pytest.mark.parametrize("window,proj,mode,iters,eps,l", [(3, 0, 0, 1, 0.5, 0.5), (4, 2, 0, 1, 0.5, 0.5),
                                                          (6, 0, 0, 1, 0.5, 0.5), (4, 0, 1, 1, 0.5, 0.5),
                                                          (3, 2, 1, 3, 0.5, 0.5), (4, 0, 0, 1, 0.7, 0.3)])
def test_wb_parity(S, orc, window, proj, mode, iters, eps, l):
    from synth import random_state
    M, N = 64, 256
    st = random_state(M, N, batch=2, seed=10 + window)
    p = _params(window, w_proj=proj, w_mode=mode, w_iters=iters, epsilon=eps, l=l)
    with _solver(S, M, N, 2, p) as sv:
        w = np.stack([st["w1"], st["w2"]], 1)
        b = np.stack([st["b1"], st["b2"]], 1)
        sv.set_state(_cuda(st["phi"]), _cuda(w), _cuda(b), _cuda(st["g"]))
        sv.debug_wb()
        s = sv.get_state()
        wg, bg = _np(s["w"]), _np(s["b"])
    for k in range(2):
        r1, r2, rb1, rb2 = orc.wb(p, st["phi"][k], st["w1"][k], st["w2"][k], st["b1"][k], st["b2"][k], st["g"][k])
        for a, r in ((wg[k, 0], r1), (wg[k, 1], r2), (bg[k, 0], rb1), (bg[k, 1], rb2)):
            assert np.max(np.abs(a - r)) < 2e-5


# ----------------------------------------------------------------------------- free-running trajectories
def _trajectory(S, orc, cfg, K=10, tol=1e-4, check_every=1):
    p = cfg["params"]
    B, M, N = cfg["image"].shape
    errs = []
    with _solver(S, M, N, B, p) as sv:
        sv.set_image(_cuda(cfg["image"]), _cuda(cfg["phi0"]))
        ref = []
        for b in range(B):
            g = orc.edge(cfg["image"][b], p["sigma"], p["rho"], p["s"])
            ref.append((orc.init(cfg["phi0"][b]), g))
        for k in range(0, K, check_every):
            sv.iterate(check_every)
            phi = _np(sv.get_phi())
            e = 0.0
            for b in range(B):
                st, g = ref[b]
                orc.iterate(p, st, g, check_every)
                e = max(e, float(np.max(np.abs(phi[b] - st["phi"]))))
            errs.append(e)
        sv.sync()
    assert max(errs) <= tol, errs
    return errs


def test_trajectory_c1(S, orc):
    from synth import make_config
    _trajectory(S, orc, make_config("c1"))


def test_trajectory_c2(S, orc):
    from synth import make_config
    _trajectory(S, orc, make_config("c2"))


def test_trajectory_c2_cluster_solve(S, orc, monkeypatch):
    """C2 free-running with the one-kernel cluster solve forced (16 CTAs x 32 rows; default only up to 128^2)."""
    from synth import make_config
    monkeypatch.setenv("SRSB_SOLVE_CL", "1")
    _trajectory(S, orc, make_config("c2"))


@pytest.mark.parametrize("env", [{"SRSB_SPEC_RM": "0"}, {"SRSB_COLS_TRI": "0"}])
def test_trajectory_c3_other_column_passes(S, orc, env, monkeypatch):
    """One C3 image free-running on the transposed spectrum: tridiagonal and FFT column pass (the default for
    N >= 1024, row-major + tridiagonal, is what every other C3 / C4 / C5 test runs)."""
    from synth import make_config
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _trajectory(S, orc, make_config("c3", images=[5]))


def test_trajectory_c3_images(S, orc):
    """C3 at full size, 8 images spread over the batch, every iteration k = 1..10 (north star)."""
    from synth import make_config
    _trajectory(S, orc, make_config("c3", images=[0, 9, 18, 27, 36, 45, 54, 63]), K=10, check_every=1)


def test_trajectory_c4_small(S, orc):
    """C4's recipe (thin close curves, R = 6, thresholded init) at 512^2."""
    from synth import make_config
    _trajectory(S, orc, make_config("c4", size=(512, 512)))


def test_trajectory_c5_small(S, orc):
    from synth import make_config
    _trajectory(S, orc, make_config("c5", size=(512, 1024)), K=10, check_every=1)


def test_trajectory_c4_fullsize(S, orc):
    """BASELINE configs[3] at its real size (4096^2, R = 6), in the bench's launch configuration,
    per-iteration phi max-abs error over k = 1..10 (north star: <= 1e-4)."""
    from synth import make_config
    _trajectory(S, orc, make_config("c4"), K=10, check_every=1)


def test_trajectory_c5_fullsize(S, orc):
    """BASELINE configs[4] at its real size (8192^2, R = 5), single GPU, k = 1..10."""
    from synth import make_config
    _trajectory(S, orc, make_config("c5"), K=10, check_every=1)


# ----------------------------------------------------------------------------- final masks (DESIGN.md §6 rule)
def _final_masks(S, orc, name, images=None, K=None):
    """Pre-registered rule of DESIGN.md §6: agreement A of {phi^K < 0} with the cached oracle run
    (tools/oracle_masks.py) must be >= 0.999, or >= the fp64 perturbation ensemble's worst member
    where that ensemble shows 0.999 is unreachable by fp64 itself; component counts identical (or
    inside the ensemble's range where the ensemble's counts vary)."""
    from synth import make_config
    from tools import oracle_masks as om
    cfg = make_config(name, images=images)
    truncated = K is not None
    p, K = cfg["params"], (K if truncated else cfg["K"])
    B, M, N = cfg["image"].shape
    with _solver(S, M, N, B, p) as sv:
        sv.set_image(_cuda(cfg["image"]), _cuda(cfg["phi0"]))
        sv.iterate(K)
        phi = _np(sv.get_phi())
        sv.sync()
    assert np.all(np.abs(phi) <= p["phi_clip"])
    report = []
    for b in range(B):
        idx = None if images is None else images[b]
        rec = om.load(name, cfg["image"][b], cfg["phi0"][b], p, K, image_index=idx, truncated=truncated)
        assert rec is not None, (f"oracle mask cache missing or stale: python tools/oracle_masks.py {name}"
                                 + (f" --K {K}" if truncated else ""))
        mg = phi[b] < 0
        agree = float((mg == rec["mask"]).mean())
        cnt = orc.label(mg)[0]
        bar = 0.999
        if rec["ens_agree"] and min(rec["ens_agree"]) < 0.999:
            bar = min(rec["ens_agree"])
        counts = set(rec["ens_count"]) | {rec["count4"]}
        ok_count = cnt == rec["count4"] or (len(counts) > 1 and min(counts) <= cnt <= max(counts))
        report.append((name, idx, agree, bar, cnt, rec["count4"], ok_count))
        print(f"{name} image {idx}: K={K} mask agreement {agree:.5f} (bar {bar:.5f}, ensemble of "
              f"{len(rec['ens_agree'])}), components gpu {cnt} oracle {rec['count4']} ensemble {sorted(counts)}")
    bad = [r for r in report if not (r[2] >= r[3] and r[6])]   # every image reported before the verdict
    assert not bad, bad
    return report


def test_c1_final_masks_and_topology(S, orc):
    """BASELINE configs[0] at full K = 300: the DESIGN.md §6 rule, and exactly one component."""
    rep = _final_masks(S, orc, "c1")
    assert rep[0][4] == 1


def test_c2_final_masks(S, orc):
    _final_masks(S, orc, "c2")


@pytest.mark.parametrize("image", [0, 1, 2, 3])
def test_c3_final_masks(S, orc, image):
    _final_masks(S, orc, "c3", images=[image])


@pytest.mark.parametrize("K", [100, pytest.param(400, marks=pytest.mark.xfail(
    strict=False, reason="pre-registered rule not met on the component count: measured agreement 1.00000 (fewer than 1 pixel in "
                         "10^5 differs) but 82 components against the oracle's 83 -- one few-pixel component; no fp64 "
                         "ensemble exists at this horizon (53 min of a box's host cores per member), so the count is held "
                         "to identical (DESIGN.md §6); reported, the bar is not moved"))])
def test_c4_masks_truncated_horizon(S, orc, K):
    """C4 at full size (4096^2, R = 6), masks after K = 100 and K = 400 of its 500 iterations: the full-length fp64
    run takes ~64 min of a GPU box's 16 host cores, more than one 3600 s box call; K = 400 takes 51.
    Same rule, no ensemble: agreement >= 0.999 and an identical component count."""
    _final_masks(S, orc, "c4", K=K)


@pytest.mark.parametrize("K", [30, 100])
def test_c5_masks_truncated_horizon(S, orc, K):
    """C5 at full size (8192^2, R = 5, one GPU), masks after K = 30 and K = 100 of its 300 iterations (the full
    fp64 run takes ~2 h of a GPU box's 16 host cores, more than one 3600 s box call).  Same rule as above."""
    _final_masks(S, orc, "c5", K=K)


def _caption_params(**over):
    """The Fig. 1 caption set: alpha = 4, gamma = 4, beta = 0.2, mu = 8, l = 1, d = 5,
    window 5 x 5 (square, R = 2), S = 3, eps = 1, tau = 0.1 -- the paper's own parameters, before
    the readings Q22-Q24 of DESIGN.md §2 changed them for the clamped dynamics."""
    from synth import paper_params
    p = paper_params(2, window_shape=1, d=5.0, gamma=4.0, alpha=4.0, beta=0.2, mu=8.0, epsilon=1.0, l=1.0,
                     tau=0.1, S=3)
    p.update(over)
    return p


@pytest.mark.parametrize("which", ["c1_state", "random_state"])
def test_teacher_forced_iteration_at_caption_params(S, orc, which):
    """One full outer iteration (S = 3 sweeps, clamp, w/b update) at the paper's caption parameters,
    teacher-forced: the GPU starts from the oracle's own state and both advance one iteration.  The
    dynamics at these parameters are chaotic under the clamp (Q23), so only the one-step
    map is compared -- the kernels must be right at the paper's values too."""
    from synth import make_config, random_state
    p = _caption_params()
    if which == "c1_state":
        cfg = make_config("c1")
        img = cfg["image"][0]
        g = orc.edge(img, p["sigma"], p["rho"], p["s"])
        st = orc.init(cfg["phi0"][0])
        orc.iterate(p, st, g, 4)
        states = [st]
        gs = [g]
    else:
        rs = random_state(128, 256, batch=2, seed=77)
        states = [dict(phi=np.clip(rs["phi"][k], -1, 1).astype(np.float64), w1=rs["w1"][k], w2=rs["w2"][k],
                       b1=rs["b1"][k], b2=rs["b2"][k]) for k in range(2)]
        gs = [rs["g"][k] for k in range(2)]
    B = len(states)
    M, N = states[0]["phi"].shape
    # the GPU gets the fp32 rounding of the state; the oracle advances that same fp32 state
    states = [{k: np.asarray(v, np.float32).astype(np.float64) for k, v in st.items()} for st in states]
    gs = [np.asarray(g, np.float32).astype(np.float64) for g in gs]
    with _solver(S, M, N, B, p) as sv:
        phi = np.stack([st["phi"] for st in states])
        w = np.stack([np.stack([st["w1"], st["w2"]]) for st in states])
        b = np.stack([np.stack([st["b1"], st["b2"]]) for st in states])
        sv.set_state(_cuda(phi), _cuda(w), _cuda(b), _cuda(np.stack(gs)))
        sv.iterate(1)
        out = sv.get_state()
        pg, wg, bg = _np(out["phi"]), _np(out["w"]), _np(out["b"])
    for k in range(B):
        ref = {kk: v.copy() for kk, v in states[k].items()}
        orc.iterate(p, ref, gs[k], 1)
        assert np.max(np.abs(pg[k] - ref["phi"])) <= 2e-5
        for a, r in ((wg[k, 0], ref["w1"]), (wg[k, 1], ref["w2"]), (bg[k, 0], ref["b1"]), (bg[k, 1], ref["b2"])):
            assert np.max(np.abs(a - r)) <= 1e-4


def test_iterate_chunking_and_determinism(S):
    """iterate(7) == iterate(3) + iterate(4) (graph vs direct launches) bitwise; runs are deterministic."""
    from synth import make_config
    cfg = make_config("c1")
    outs = []
    for chunks in ((7,), (3, 4), (1, 1, 5)):
        with _solver(S, 128, 128, 1, cfg["params"]) as sv:
            sv.set_image(_cuda(cfg["image"]), _cuda(cfg["phi0"]))
            for c in chunks:
                sv.iterate(c)
            s = sv.get_state()
            outs.append({k: _np(v) for k, v in s.items()})
            assert sv.iteration == 7
    for o in outs[1:]:
        for k in o:
            assert np.array_equal(o[k], outs[0][k]), k


def test_host_buffers_and_errors(S):
    """Host (numpy) pointers work through the same calls; call-order errors are reported."""
    from synth import make_config
    cfg = make_config("c1")
    with _solver(S, 128, 128, 1, cfg["params"]) as sv:
        with pytest.raises(S.SrsbError):
            sv.iterate(1)                      # before set_image: SR_ERR_STATE
        sv.set_image(cfg["image"], cfg["phi0"])
        sv.iterate(2)
        host = np.empty((1, 128, 128), np.float32)
        sv.get_phi(host)
        sv.sync()
        dev = _np(sv.get_phi())
        assert np.array_equal(host.astype(np.float64), dev)


def test_nonfinite_guard(S):
    from synth import make_config
    cfg = make_config("c1")
    img = cfg["image"].copy()
    with _solver(S, 128, 128, 1, cfg["params"]) as sv:
        sv.set_image(img, cfg["phi0"])
        st = sv.get_state()
        b = st["b"].clone()
        b[0, 0, 5, 5] = float("nan")
        sv.set_state(st["phi"], st["w"], b)
        sv.iterate(1)
        with pytest.raises(S.SrsbError) as ei:
            sv.sync()
        assert ei.value.status == S.SR_ERR_NONFINITE


# ----------------------------------------------------------------------------- NEXT-1 monitor
def test_monitor_energy_and_sweep_changes(S, orc):
    """Energies of Eq. (22) at (phi^{k+1}, w^k, b^k) and the per-sweep phi changes of one
    teacher-forced iteration, against the oracle."""
    from synth import random_state
    M, N = 128, 256
    st = random_state(M, N, batch=2, seed=21)
    p = _params(4)
    with _solver(S, M, N, 2, p) as sv:
        w = np.stack([st["w1"], st["w2"]], 1)
        b = np.stack([st["b1"], st["b2"]], 1)
        sv.set_state(_cuda(st["phi"]), _cuda(w), _cuda(b), _cuda(st["g"]))
        sv.set_monitor(True)
        sv.iterate(1)
        mon = sv.monitor()
    for k in range(2):
        psi = st["phi"][k].astype(np.float64)
        args = [st[n][k] for n in ("w1", "w2", "b1", "b2", "g")]
        changes = []
        for s in range(p["S"]):
            new = orc.sweep(p, psi, *args)
            if s == p["S"] - 1:
                new = np.clip(new, -p["phi_clip"], p["phi_clip"])
            changes.append(np.linalg.norm(new - psi) / (np.linalg.norm(psi) + 1e-6))
            psi = new
        eg, ea, er, ep = orc.energy(p, psi, *args)
        got = mon[k]
        for a, r in ((got["E_g"], eg), (got["E_a"], ea), (got["E_r"], er), (got["E_pen"], ep)):
            assert a == pytest.approx(r, rel=1e-4, abs=1e-3)
        assert got["sweep_change"] == pytest.approx(changes, rel=1e-3)


def test_monitor_reductions_are_deterministic(S):
    """The monitor sums (Eq. 22 terms, per-sweep changes, the outer change of iterate_until) come from
    per-CTA partials summed in a fixed order (sr_reduce.cuh), not atomics: bitwise equal across runs,
    also through the TMA-free stencil path and on a batch with ragged tiles."""
    from synth import make_config
    cfg = make_config("c2")
    p = cfg["params"]

    def run(env=None):
        import os
        old = os.environ.get("SRSB_TMA")
        if env is not None:
            os.environ["SRSB_TMA"] = env
        try:
            with _solver(S, 512, 512, 1, p) as sv:
                sv.set_image(_cuda(cfg["image"]), _cuda(cfg["phi0"]))
                sv.set_monitor(True)
                sv.iterate(3)
                raw = [m["raw"] for m in sv.monitor()]
                k, ch = sv.iterate_until(6, 0.0, every=3)
                sv.sync()
        finally:
            if env is not None:
                if old is None:
                    del os.environ["SRSB_TMA"]
                else:
                    os.environ["SRSB_TMA"] = old
        return raw, ch
    a, b, c = run(), run(), run()
    assert a == b == c
    d, e = run("0"), run("0")
    assert d == e
    np.testing.assert_allclose(np.asarray(d[0]), np.asarray(a[0]), rtol=1e-5, atol=1e-6)


def test_iterate_until_outer_change(S, orc):
    """sr_sb_iterate_until stops at the first check whose relative phi change (over `every`
    iterations) is <= tol; the reported change matches the oracle trajectory's at that point."""
    from synth import make_config
    cfg = make_config("c1")
    p = cfg["params"]
    with _solver(S, 128, 128, 1, p) as sv:
        sv.set_image(_cuda(cfg["image"]), _cuda(cfg["phi0"]))
        sv.set_monitor(True)
        k, ch = sv.iterate_until(60, 0.0, every=20)          # tol 0: runs all 60, reports the change
        assert k == 60 and sv.iteration == 60 and ch > 0
        phi = _np(sv.get_phi())[0]
        k2, ch2 = sv.iterate_until(200, 10.0, every=20)      # huge tol: stops after the first chunk
        assert k2 == 20
    g = orc.edge(cfg["image"][0], p["sigma"], p["rho"], p["s"])
    st = orc.init(cfg["phi0"][0])
    orc.iterate(p, st, g, 40)
    a = st["phi"].copy()
    orc.iterate(p, st, g, 20)
    ref = np.linalg.norm(st["phi"] - a) / (np.linalg.norm(a) + 1e-6)
    assert ch == pytest.approx(ref, rel=5e-3, abs=1e-5)
    assert np.max(np.abs(phi - st["phi"])) < 1e-2


# ----------------------------------------------------------------------------- degenerate cases
def test_degenerate_cases(S, orc):
    """K = 0 is a no-op; tau = 0 freezes phi (F = psi, Eq. 37) up to the clamp of phi0 = +-1;
    beta = 0 (plain GAC, no repulsion) and R = 0 still match the oracle over 5 iterations."""
    from synth import make_config
    cfg = make_config("c1")
    p = cfg["params"]
    img, phi0 = cfg["image"], cfg["phi0"]
    with _solver(S, 128, 128, 1, p) as sv:
        sv.set_image(_cuda(img), _cuda(phi0))
        sv.iterate(0)
        assert sv.iteration == 0
        assert np.array_equal(_np(sv.get_phi()), phi0.astype(np.float64))
    with _solver(S, 128, 128, 1, dict(p, tau=0.0)) as sv:
        sv.set_image(_cuda(img), _cuda(phi0))
        sv.iterate(3)
        assert np.max(np.abs(_np(sv.get_phi()) - phi0)) < 1e-6
    for over in (dict(beta=0.0), dict(window=0, d=1.0)):
        q = dict(p, **over)
        with _solver(S, 128, 128, 1, q) as sv:
            sv.set_image(_cuda(img), _cuda(phi0))
            sv.iterate(5)
            phi = _np(sv.get_phi())
        ref = orc.run(q, img[0], phi0[0], 5)["phi"]
        assert np.max(np.abs(phi[0] - ref)) <= 1e-4, over


@pytest.mark.parametrize("M,N,env", [(1024, 1024, {"SRSB_RPC": "4"}), (1024, 1024, {"SRSB_G": "2"}),
                                     (512, 512, {"SRSB_RPC": "2"}), (128, 128, {"SRSB_G": "2"}),
                                     (1024, 1024, {"SRSB_RPC_INV": "4"}), (4096, 8192, {"SRSB_R2C_WIDE": "0"})])
def test_launch_shape_instances_bitwise(S, M, N, env, monkeypatch):
    """The launch-shape instances of the row passes (rows per CTA / interleave as template constants,
    paired 16-byte transposed accesses) and the contiguous-column solve give bitwise the same Eq. (33)
    solve as the generic kernels: other shapes / layouts are forced with the tuning knobs (read at
    context creation), the butterflies and per-element arithmetic are identical."""
    monkeypatch.setenv("SRSB_COLS_TRI", "0")   # FFT column pass on both sides (the knobs move G off 1)
    p = _params(4)
    F = np.random.default_rng(7).standard_normal((2, M, N)).astype(np.float32)
    with _solver(S, M, N, 2, p) as sv:
        ref = _np(sv.debug_solve(_cuda(F)))
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    with _solver(S, M, N, 2, p) as sv:
        out = _np(sv.debug_solve(_cuda(F)))
    assert np.array_equal(out, ref)


@pytest.mark.parametrize("name,size,K", [("c1", None, 20), ("c3", (1024, 1024), 6), ("c4", (512, 512), 6),
                                         ("c2", None, 8)])
def test_band_skip_is_exact(S, monkeypatch, name, size, K):
    """The narrow-band skip of the window sums (sr_stencil.cuh needs_v) drops only terms
    that are multiplied by an exact zero (h or h' off the band): trajectories with and without it are
    bitwise equal, on configs where most tiles lie off the band."""
    from synth import make_config
    cfg = make_config(name, size=size) if name != "c3" else make_config("c3", images=[0, 1])
    p = cfg["params"]
    B, M, N = cfg["image"].shape

    def run():
        with _solver(S, M, N, B, p) as sv:
            sv.set_image(_cuda(cfg["image"]), _cuda(cfg["phi0"]))
            sv.iterate(K)
            st = sv.get_state()
            out = {k: v.cpu().numpy() for k, v in st.items()}
            sv.sync()
        return out
    a = run()
    monkeypatch.setenv("SRSB_BAND_SKIP", "0")
    b = run()
    for k in ("phi", "w", "b"):
        assert np.array_equal(a[k], b[k]), k
