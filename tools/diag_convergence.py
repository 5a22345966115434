"""Print the monitor's last-sweep relative phi change and E_total every `every` iterations."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from synth import make_config
from paper_2003_12693_b200 import Solver
name = sys.argv[1] if len(sys.argv) > 1 else "c1"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
every = int(sys.argv[3]) if len(sys.argv) > 3 else 100
c = make_config(name) if name != "c3" else make_config("c3", images=[0])
p = c["params"]
_, M, N = c["image"].shape
keys = ("gamma", "alpha", "beta", "mu", "epsilon", "l", "d", "window_shape", "tau", "S", "rho", "sigma", "s",
        "phi_clip", "w_proj", "w_mode", "w_iters")
sv = Solver(M, N, 1, window=p["window"], **{k: p[k] for k in keys})
sv.set_image(torch.from_numpy(c["image"][:1]).cuda(), torch.from_numpy(c["phi0"][:1]).cuda())
sv.set_monitor(True)
for k in range(0, K, every):
    sv.iterate(every)
    m = sv.monitor()[0]
    inside = (sv.get_phi() < 0).float().mean().item()
    print(f"k={k + every:5d} change={m['sweep_change'][-1]:.3e} E={m['E_total']:.4f} inside={inside:.4f}", flush=True)
