"""Synthetic 3-D workload for the NEXT-3 extension (Fig. 6: a CT volume, not available).

A seeded stand-in with the structure of the paper's 3-D case: a few solid, possibly touching
ellipsoids (bone-like blobs at intensity U(0.6, 1)) on a 0 background plus Gaussian noise; phi0 =
+1 except a border (BASELINE convention), returned negated to the paper's convention (phi < 0
inside, Eq. 3).  Arrays are float32 [D][M][N].  Nothing here implements a step of the method.
"""
from __future__ import annotations

import math

import numpy as np

from .configs import BASE_SEED, paper_params

V3_DEFAULT = (128, 128, 128)


def ball_weight_sum(window: int, d: float, shape: int = 0) -> float:
    """sum over the ball (shape 0) or cube (1) of radius `window` of exp(-(p^2+q^2+r^2)/d^2)."""
    s = 0.0
    for r in range(-window, window + 1):
        for p in range(-window, window + 1):
            for q in range(-window, window + 1):
                if shape == 0 and p * p + q * q + r * r > window * window:
                    continue
                s += math.exp(-(p * p + q * q + r * r) / (d * d))
    return s


def paper_params3(window: int, **over) -> dict:
    """The 2-D design parameter set (synth.paper_params) with Q24's repulsion normalisation taken
    over the 3-D ball: beta * G_ball = 0.2 * G(5x5 square, d = 5) (reading Q26)."""
    d = float(over.get("d", window if window > 0 else 1.0))
    shape = int(over.get("window_shape", 0))
    p = paper_params(window, **over)
    if "beta" not in over:
        from .configs import window_weight_sum
        p["beta"] = 0.2 * window_weight_sum(2, 5.0, 1) / ball_weight_sum(window, d, shape)
    return p


def make_volume(size=V3_DEFAULT, n=12, window=3, seed=0, noise=0.15, border=4) -> dict:
    D, M, N = size
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([BASE_SEED, 300, seed, D, M, N])))
    z, i, j = np.meshgrid(np.arange(D, dtype=np.float64), np.arange(M, dtype=np.float64),
                          np.arange(N, dtype=np.float64), indexing="ij")
    vol = np.zeros((D, M, N), dtype=np.float64)
    smin = 0.06 * min(D, M, N)
    smax = 0.22 * min(D, M, N)
    for _ in range(n):
        c = [rng.uniform(0.2 * s, 0.8 * s) for s in (D, M, N)]
        a = rng.uniform(smin, smax, 3)
        # random orientation: rotate the offsets by a random orthogonal matrix (QR of a Gaussian)
        Q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
        off = np.stack([z - c[0], i - c[1], j - c[2]], -1) @ Q
        inside = (off[..., 0] / a[0]) ** 2 + (off[..., 1] / a[1]) ** 2 + (off[..., 2] / a[2]) ** 2 <= 1.0
        vol[inside] = rng.uniform(0.6, 1.0)
    vol += noise * rng.standard_normal(vol.shape)
    phi_bj = -np.ones((D, M, N))
    phi_bj[border:D - border, border:M - border, border:N - border] = 1.0
    return {"volume": vol.astype(np.float32), "phi0": (-phi_bj).astype(np.float32),
            "params": paper_params3(window), "window": window}
