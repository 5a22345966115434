"""Diagnostic (GPU only, no oracle): how sensitive are the final masks of a config to fp32-sized
noise?  Runs the config once, and `members` more times with phi^1 + U(-1e-7, 1e-7) (seeded), all in
fp32 on the GPU, and prints the mask agreement of each member with the unperturbed run.  This is a
proxy for the fp64 ensemble of tools/oracle_masks.py (which is what the parity rule uses); it
tells whether a full-length fp64 ensemble is worth its CPU hours for a config.

    python tools/gpu_mask_spread.py c5 --members 2
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--members", type=int, default=2)
    ap.add_argument("--images", type=int, nargs="*", default=None)
    a = ap.parse_args()
    from paper_2003_12693_b200 import srsb as S
    from synth import make_config
    cfg = make_config(a.config, images=a.images)
    p, K = cfg["params"], cfg["K"]
    B, M, N = cfg["image"].shape
    keys = ("gamma", "alpha", "beta", "mu", "epsilon", "l", "d", "window_shape", "tau", "S", "rho", "sigma",
            "s", "phi_clip", "w_proj", "w_mode", "w_iters")
    t0 = time.time()
    with S.Solver(M, N, B, window=p["window"], **{k: p[k] for k in keys}) as sv:
        sv.set_image(torch.from_numpy(cfg["image"]).cuda(), torch.from_numpy(cfg["phi0"]).cuda())
        sv.iterate(1)
        st1 = {k: v.clone() for k, v in sv.get_state().items()}
        sv.iterate(K - 1)
        base = sv.get_phi().cpu().numpy() < 0
        out = []
        for m in range(1, a.members + 1):
            rng = np.random.default_rng(1000 + m)
            phi = st1["phi"].cpu().numpy() + rng.uniform(-1e-7, 1e-7, st1["phi"].shape).astype(np.float32)
            sv.set_state(torch.from_numpy(phi.astype(np.float32)).cuda(), st1["w"], st1["b"], st1["g"])
            sv.iterate(K - 1)
            mm = sv.get_phi().cpu().numpy() < 0
            out.append([float((mm[b] == base[b]).mean()) for b in range(B)])
        sv.sync()
    print(json.dumps({"config": a.config, "images": a.images, "K": K, "agreement": out,
                      "min": float(np.min(out)), "seconds": time.time() - t0}))


if __name__ == "__main__":
    main()
