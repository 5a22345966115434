"""Diagnostic: run one RHS launch for every window radius 0..8 and both shapes on a random state,
compare with the oracle; prints max relative error per (R, shape).  python tools/diag_windows.py [M N]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (diagnostic tool: test infrastructure)
from paper_2003_12693_b200 import Solver  # noqa: E402
from synth import paper_params, random_state  # noqa: E402

KEYS = ("gamma", "alpha", "beta", "mu", "epsilon", "l", "d", "window_shape", "tau", "S", "rho", "sigma", "s",
        "phi_clip", "w_proj", "w_mode", "w_iters")

M, N = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (128, 256)
ONLY = [int(x) for x in os.environ.get("DIAG_R", "").split(",") if x]
for R in ONLY or range(9):
    for shape in (0, 1):
        p = paper_params(R, window_shape=shape, phi_solver=int(os.environ.get("DIAG_AOS", "1")))
        st = random_state(M, N, batch=1, seed=R)
        try:
            with Solver(M, N, 1, window=R, phi_solver=p["phi_solver"], **{k: p[k] for k in KEYS}) as sv:
                w = np.stack([st["w1"], st["w2"]], 1)
                b = np.stack([st["b1"], st["b2"]], 1)
                c = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
                sv.set_state(c(st["phi"]), c(w), c(b), c(st["g"]))
                F = sv.debug_rhs().cpu().numpy().astype(np.float64)
            ref = oracle.rhs(p, st["phi"][0], st["w1"][0], st["w2"][0], st["b1"][0], st["b2"][0], st["g"][0])
            print(R, shape, f"{np.max(np.abs(F[0] - ref) / (1 + np.abs(ref))):.2e}", flush=True)
        except Exception as e:
            print(R, shape, "ERROR", str(e)[:120], flush=True)
            sys.exit(1)
