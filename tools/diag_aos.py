"""Diagnostic: per-iteration max |phi_gpu - phi_oracle| for the FFT and AOS phi solvers on one
config (free-running), to separate kernel error from the dynamics' amplification of rounding.

    python tools/diag_aos.py c2 20
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (diagnostic tool: test infrastructure)
from paper_2003_12693_b200 import Solver  # noqa: E402
from synth import make_config  # noqa: E402

KEYS = ("gamma", "alpha", "beta", "mu", "epsilon", "l", "d", "window_shape", "tau", "S", "rho", "sigma", "s",
        "phi_clip", "w_proj", "w_mode", "w_iters")


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    c = make_config(name)
    B, M, N = c["image"].shape
    for solver in (0, 1):
        p = dict(c["params"], phi_solver=solver)
        g = oracle.edge(c["image"][0], p["sigma"], p["rho"], p["s"])
        st = oracle.init(c["phi0"][0])
        errs = []
        with Solver(M, N, 1, window=p["window"], phi_solver=solver, **{k: p[k] for k in KEYS}) as sv:
            sv.set_image(torch.from_numpy(c["image"][:1]).cuda(), torch.from_numpy(c["phi0"][:1]).cuda())
            for k in range(K):
                sv.iterate(1)
                phi = sv.get_phi().cpu().numpy().astype(np.float64)[0]
                oracle.iterate(p, st, g, 1)
                errs.append(float(np.max(np.abs(phi - st["phi"]))))
        print(["fft", "aos"][solver], " ".join(f"{e:.2e}" for e in errs), flush=True)


if __name__ == "__main__":
    main()
