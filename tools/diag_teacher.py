"""Teacher-forced one-step diagnostic: for k = 1..K, load the oracle's state k-1 into
the GPU context, run ONE iteration on the GPU, and report max |GPU - oracle| of phi, w, b at step k.
Separates per-step kernel error from trajectory amplification.  Test tooling (uses oracle/)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import oracle as O
from synth import make_config
from paper_2003_12693_b200 import Solver

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
size = tuple(int(x) for x in sys.argv[3].split("x")) if len(sys.argv) > 3 else None
c = make_config(name, size=size) if size else (make_config(name, images=[0]) if name == "c3" else make_config(name))
p = c["params"]
M, N = c["image"].shape[1:]
keys = ("gamma", "alpha", "beta", "mu", "epsilon", "l", "d", "window_shape", "tau", "S", "rho", "sigma", "s",
        "phi_clip", "w_proj", "w_mode", "w_iters")
sv = Solver(M, N, 1, window=p["window"], **{k: p[k] for k in keys})
sv.set_image(torch.from_numpy(c["image"][:1]).cuda(), torch.from_numpy(c["phi0"][:1]).cuda())
g_gpu = sv.get_state()["g"]
g = O.edge(c["image"][0], p["sigma"], p["rho"], p["s"])
st = O.init(c["phi0"][0])
free = Solver(M, N, 1, window=p["window"], **{k: p[k] for k in keys})
free.set_image(torch.from_numpy(c["image"][:1]).cuda(), torch.from_numpy(c["phi0"][:1]).cuda())
f32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
for k in range(1, K + 1):
    w = np.stack([st["w1"], st["w2"]])[None]
    b = np.stack([st["b1"], st["b2"]])[None]
    sv.set_state(f32(st["phi"][None]), f32(w), f32(b), g_gpu)
    sv.iterate(1)
    s = {kk: v.cpu().numpy().astype(np.float64) for kk, v in sv.get_state().items()}
    O.iterate(p, st, g, 1)
    free.iterate(1)
    fphi = free.get_phi().cpu().numpy()[0].astype(np.float64)
    e_phi = np.abs(s["phi"][0] - st["phi"])
    i = np.unravel_index(e_phi.argmax(), e_phi.shape)
    print(f"k={k:3d} one-step: phi {e_phi.max():.2e} at {i} (orc {st['phi'][i]:+.4f}) "
          f"w {max(np.abs(s['w'][0,0]-st['w1']).max(), np.abs(s['w'][0,1]-st['w2']).max()):.2e} "
          f"b {max(np.abs(s['b'][0,0]-st['b1']).max(), np.abs(s['b'][0,1]-st['b2']).max()):.2e} | free-run phi "
          f"{np.abs(fphi - st['phi']).max():.2e}", flush=True)
