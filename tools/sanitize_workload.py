"""Small workload that launches every kernel of libsrsb.so once or a few times, for
compute-sanitizer (SURVEY.md §4b tier T5; tools/run_sanitizers.sh):

  * C1 (128^2, R = 3) and C2 (512^2, R = 4): set_image (blur / edge / init), 2 iterations through the
    captured CUDA graph and 1 by direct launches -- the TMA stencils (k_rhs_tma, k_wb_tma: mbarriers,
    cp.async.bulk.tensor, L2 prefetch), the row / column FFT passes;
  * the same with the monitor on (energy and sweep-change reductions), the fixed-point w mode, the
    square window, l != eps (the general regularizer branch) and the non-TMA stencils (SRSB_TMA=0);
  * a P = 2 slab group (halo copies, the chunked all-to-all on the comm stream, the slab graph);
  * the AOS phi solver (NEXT-4) and one small 3-D volume (NEXT-3).

No oracle: this only drives the kernels.  Exits non-zero if any call reports an error.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

KEYS = ("gamma", "alpha", "beta", "mu", "epsilon", "l", "d", "window_shape", "tau", "S", "rho", "sigma", "s",
        "phi_clip", "w_proj", "w_mode", "w_iters")


def run(S, cfg, K=3, monitor=False, slabs=None, **over):
    p = dict(cfg["params"])
    p.update(over)
    B, M, N = cfg["image"].shape
    kw = {k: p[k] for k in KEYS}
    if "phi_solver" in over:
        kw["phi_solver"] = over["phi_solver"]
    with S.Solver(M, N, B if slabs is None else 1, window=p["window"], slabs=slabs, **kw) as sv:
        sv.set_image(torch.from_numpy(cfg["image"][: (B if slabs is None else 1)]).cuda(),
                     torch.from_numpy(cfg["phi0"][: (B if slabs is None else 1)]).cuda())
        if monitor:
            sv.set_monitor(True)
        sv.iterate(2)
        sv.iterate(1)
        if monitor:
            sv.monitor()
        phi = sv.get_phi()
        sv.sync()
    assert torch.isfinite(phi).all()
    return phi


def main():
    from paper_2003_12693_b200 import srsb as S
    from synth import make_config
    from synth.volumes import make_volume
    torch.cuda.set_device(0)
    which = sys.argv[1:] or ["c1", "c2", "modes", "slab", "aos", "v3d"]
    c1, c2 = make_config("c1"), make_config("c2")
    if "c1" in which:
        run(S, c1)
    if "c2" in which:
        run(S, c2, K=2)
    if "modes" in which:
        run(S, c1, monitor=True)
        run(S, c1, w_mode=1, w_iters=2)
        run(S, c1, window_shape=1)
        run(S, c1, epsilon=0.5, l=1.0)
        os.environ["SRSB_TMA"] = "0"
        run(S, c1)
        del os.environ["SRSB_TMA"]
    if "slab" in which:
        run(S, make_config("c5", size=(256, 256)), slabs=2)
    if "aos" in which:
        run(S, c1, phi_solver=1)
    if "v3d" in which:
        v = make_volume(size=(16, 32, 32), window=2)
        p = v["params"]
        with S.Solver3(16, 32, 32, window=2, **{k: p[k] for k in KEYS if k in p}) as sv:
            sv.set_image(torch.from_numpy(v["volume"]).cuda(), torch.from_numpy(v["phi0"]).cuda())
            sv.iterate(2)
            phi = sv.get_phi()
            sv.sync()
        assert torch.isfinite(phi).all()
    torch.cuda.synchronize()
    print("sanitize workload OK:", " ".join(which))


if __name__ == "__main__":
    main()
