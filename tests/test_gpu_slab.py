"""Slab decomposition (BASELINE configs[4]) on one GPU.

P row slabs of one image, with the halo exchanges and the all-to-all spectrum transpose done as
device copies between the P slab contexts of this process (sr_sb_create_slab_group), run the same
per-row / per-column butterflies and per-pixel stencils as the whole-image context, so the result
must be BITWISE identical to P = 1.  The NCCL backend is exercised with a one-rank communicator
(its wrap rows are local copies; the all-to-all is NCCL's).  Multi-GPU NCCL runs need >1 GPU and
are not part of this single-GPU suite.
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
    assert torch.cuda.is_available()
    return srsb


@pytest.fixture(autouse=True, params=["tri", "fft"])
def _column_pass(request, monkeypatch):
    """The bitwise slab == whole-image property is a statement about identical arithmetic in identical order,
    so both sides run the same column pass (knobs read at context creation): 'tri' = the cyclic tridiagonal
    solve on the transposed spectrum with contiguous columns (slab contexts: column segments of the
    all-to-all receive buffer; whole image: G = 1, no row-major spectrum, no cluster solve), 'fft' = FFT ->
    divide by the symbol -> inverse FFT on both."""
    if request.param == "fft":
        monkeypatch.setenv("SRSB_COLS_TRI", "0")
    else:
        monkeypatch.setenv("SRSB_SPEC_RM", "0")
        monkeypatch.setenv("SRSB_SOLVE_CL", "0")
        monkeypatch.setenv("SRSB_G", "1")
    return request.param


KEYS = ("gamma", "alpha", "beta", "mu", "epsilon", "l", "d", "window_shape", "tau", "S", "rho", "sigma", "s",
        "phi_clip", "w_proj", "w_mode", "w_iters")


def _run(S, cfg, K, **kw):
    p = cfg["params"]
    _, M, N = cfg["image"].shape
    with S.Solver(M, N, 1, window=p["window"], **{k: p[k] for k in KEYS}, **kw) as sv:
        img = torch.from_numpy(cfg["image"][:1]).cuda()
        phi0 = torch.from_numpy(cfg["phi0"][:1]).cuda()
        if sv.M_local != M:                         # NCCL slab: local rows only
            r0 = 0
            img, phi0 = img[:, r0:r0 + sv.M_local].contiguous(), phi0[:, r0:r0 + sv.M_local].contiguous()
        sv.set_image(img, phi0)
        g = sv.get_state(fields=("g",))["g"].cpu().numpy()
        sv.iterate(K)
        phi = sv.get_phi().cpu().numpy()
        sv.sync()
    return phi, g


@pytest.mark.parametrize("name,size,P,K", [("c1", None, 2, 6), ("c1", None, 4, 3), ("c5", (512, 512), 2, 5),
                                           ("c5", (512, 512), 8, 4), ("c3", (256, 256), 4, 5), ("c4", (256, 512), 2, 4)])
def test_slab_group_bitwise_equals_whole_image(S, name, size, P, K):
    from synth import make_config
    cfg = make_config(name, size=size) if size else make_config(name)
    if name == "c3":
        cfg = make_config("c3", images=[0], size=size)
    ref_phi, ref_g = _run(S, cfg, K)
    phi, g = _run(S, cfg, K, slabs=P)
    assert np.array_equal(g, ref_g)
    assert np.array_equal(phi, ref_phi), np.abs(phi - ref_phi).max()


def test_slab_group_fixed_point_and_square_window(S):
    from synth import make_config
    cfg = make_config("c1")
    cfg["params"] = dict(cfg["params"], w_mode=1, w_iters=2, window_shape=1)
    ref_phi, _ = _run(S, cfg, 3)
    phi, _ = _run(S, cfg, 3, slabs=4)
    assert np.array_equal(phi, ref_phi)


def test_slab_nccl_one_rank(S):
    from synth import make_config
    cfg = make_config("c5", size=(256, 256))
    ref_phi, ref_g = _run(S, cfg, 4)
    ident = S.nccl_unique_id()
    phi, g = _run(S, cfg, 4, nccl=(1, 0, ident))
    assert np.array_equal(g, ref_g)
    assert np.array_equal(phi, ref_phi)


@pytest.mark.parametrize("chunks,graph", [("1", "1"), ("2", "1"), ("4", "1"), ("4", "0"), ("8", "1")])
def test_slab_chunked_alltoall_and_graph_bitwise(S, chunks, graph, monkeypatch):
    """The pipelined transpose (all-to-all chunk k+1 on the comm stream while the column solve of
    chunk k runs) and the CUDA graph of the slab iteration (kernels + exchanges +
    fork/join) change no arithmetic: bitwise equal to the whole image, odd and even K."""
    from synth import make_config
    cfg = make_config("c5", size=(512, 512))
    ref_phi, _ = _run(S, cfg, 5)
    monkeypatch.setenv("SRSB_A2A_CHUNKS", chunks)
    monkeypatch.setenv("SRSB_GRAPH", graph)
    phi, _ = _run(S, cfg, 5, slabs=4)
    assert np.array_equal(phi, ref_phi)
    p = cfg["params"]
    with S.Solver(512, 512, 1, window=p["window"], **{k: p[k] for k in KEYS}, slabs=4) as sv:
        assert sv.a2a_chunks == int(chunks)


def test_slab_nccl_one_rank_graph_and_chunks(S, monkeypatch):
    """The NCCL backend's op lists (self pairs on a one-rank communicator) under the graph and the
    chunked transpose: bitwise equal to the whole image."""
    from synth import make_config
    cfg = make_config("c5", size=(256, 256))
    ref_phi, _ = _run(S, cfg, 4)
    monkeypatch.setenv("SRSB_A2A_CHUNKS", "4")
    phi, _ = _run(S, cfg, 4, nccl=(1, 0, S.nccl_unique_id()))
    assert np.array_equal(phi, ref_phi)


def test_slab_validation(S):
    from synth import make_config
    cfg = make_config("c1")
    p = cfg["params"]
    with pytest.raises(S.SrsbError):
        S.Solver(128, 128, 2, window=3, slabs=2)                 # batch must be 1
    with pytest.raises(S.SrsbError):
        S.Solver(128, 128, 1, window=3, slabs=32)                # 4 local rows < 8
    with pytest.raises(S.SrsbError):
        S.Solver(128, 128, 1, window=3, slabs=3)                 # not a power of two
    del p


def test_dist_solver_on_one_rank_nccl_group(S):
    """srsb.DistSolver with default arguments on an NCCL process group (the group bench.py uses): the
    unique id is broadcast as a device tensor (NCCL has no CPU tensors), then the one-rank slab
    context runs bitwise like the whole image."""
    import socket
    import torch.distributed as dist
    from synth import make_config
    cfg = make_config("c5", size=(256, 256))
    ref_phi, _ = _run(S, cfg, 4)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", world_size=1, rank=0)
    try:
        p = cfg["params"]
        with S.DistSolver(256, 256, window=p["window"], **{k: p[k] for k in KEYS}) as sv:
            sv.set_image(torch.from_numpy(cfg["image"]).cuda(), torch.from_numpy(cfg["phi0"]).cuda())
            sv.iterate(4)
            phi = sv.get_phi().cpu().numpy()
            sv.sync()
    finally:
        dist.destroy_process_group()
    assert np.array_equal(phi, ref_phi)
