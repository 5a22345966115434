"""Cache of full-length oracle runs: final masks {phi < 0} of the BASELINE configs, bit-packed.

    python tools/oracle_masks.py c2 --ensemble 8
    python tools/oracle_masks.py c3 --images 0 1 2 3
    python tools/oracle_masks.py c5 --K 30      (a truncated horizon: see DESIGN.md §6)

Calls ONLY `oracle/` (the float64 C oracle) and `synth/` (seeded inputs); nothing here touches
the CUDA path, so every stored value comes from the oracle (task rule: a stored value is written
by a committed script that calls only oracle/).  Output: tests/golden/masks/<cfg>[_i<img>].npz with

  key      sha256 of (image, phi0, params, K, ORACLE_RUN_VERSION): the GPU test recomputes it from
           synth and refuses a stale file (it fails, it does not skip);
  packed   np.packbits of the final mask {phi^K < 0} (reading Q19: phi = 0 is outside);
  count4   4-connected components of the mask (Q18), by orc.label;
  ens_agree / ens_count
           the perturbation ensemble (pre-registered rule): member m continues the
           SAME oracle run from phi^1 + U(-1e-7, 1e-7) (seeded per member; fp32-sized noise: the
           fp32 spacing at 1 is 1.19e-7) for the remaining K - 1 iterations; its mask agreement with
           the unperturbed run and its component count;
  wall_s, threads  how long the oracle took, on how many OpenMP threads.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

OUT = os.path.join(ROOT, "tests", "golden", "masks")
ORACLE_RUN_VERSION = "orc-r2-1"   # bump when the oracle's arithmetic changes (commit must cite why)
PERTURB = 1e-7


def run_key(image: np.ndarray, phi0: np.ndarray, params: dict, K: int) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(image, dtype=np.float32).tobytes())
    h.update(np.ascontiguousarray(phi0, dtype=np.float32).tobytes())
    h.update(json.dumps({k: params[k] for k in sorted(params)}, sort_keys=True).encode())
    h.update(f"K={K};{ORACLE_RUN_VERSION}".encode())
    return h.hexdigest()


def cache_path(name: str, image_index: int | None = None, K: int | None = None) -> str:
    """K: a truncated horizon (records of the full-K run carry no suffix)."""
    stem = name if image_index is None else f"{name}_i{image_index}"
    return os.path.join(OUT, stem + (f"_k{K}" if K is not None else "") + ".npz")


def load(name: str, image: np.ndarray, phi0: np.ndarray, params: dict, K: int, image_index=None,
         truncated: bool = False) -> dict | None:
    """The cached record for this exact input, or None when it is missing or stale."""
    p = cache_path(name, image_index, K if truncated else None)
    if not os.path.exists(p):
        return None
    z = np.load(p)
    if str(z["key"]) != run_key(image, phi0, params, K):
        return None
    shape = tuple(int(x) for x in z["shape"])
    mask = np.unpackbits(z["packed"])[: shape[0] * shape[1]].reshape(shape).astype(bool)
    rec = dict(mask=mask, count4=int(z["count4"]), K=int(z["K"]))
    rec["ens_agree"] = [float(x) for x in z["ens_agree"]]
    rec["ens_count"] = [int(x) for x in z["ens_count"]]
    return rec


def compute(name: str, image_index: int | None, ensemble: int, log=print, out_dir: str | None = None,
            K_override: int | None = None) -> str:
    import oracle as orc
    from synth import make_config

    cfg = make_config(name, images=None if image_index is None else [image_index])
    p, K = cfg["params"], cfg["K"] if K_override is None else K_override
    img, phi0 = cfg["image"][0], cfg["phi0"][0]
    key = run_key(img, phi0, p, K)
    t0 = time.time()
    g = orc.edge(img, p["sigma"], p["rho"], p["s"])
    st1 = orc.init(phi0)
    orc.iterate(p, st1, g, 1)
    base = {k: v.copy() for k, v in st1.items()}
    orc.iterate(p, base, g, K - 1)
    mask = base["phi"] < 0
    count = orc.label(mask)[0]
    log(f"{name} img={image_index} base done in {time.time() - t0:.0f} s: count4={count}")
    agree, counts = [], []
    for m in range(1, ensemble + 1):
        rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([12693, 777, int(name[1:]),
                                                                         image_index or 0, m])))
        st = {k: v.copy() for k, v in st1.items()}
        st["phi"] = st["phi"] + rng.uniform(-PERTURB, PERTURB, st["phi"].shape)
        orc.iterate(p, st, g, K - 1)
        mm = st["phi"] < 0
        agree.append(float((mm == mask).mean()))
        counts.append(int(orc.label(mm)[0]))
        log(f"  member {m}: agreement {agree[-1]:.6f} count4 {counts[-1]} ({time.time() - t0:.0f} s)")
    os.makedirs(out_dir or OUT, exist_ok=True)
    path = cache_path(name, image_index, K_override)
    if out_dir:
        path = os.path.join(out_dir, os.path.basename(path))
    np.savez_compressed(path, key=np.array(key), shape=np.array(mask.shape), packed=np.packbits(mask.ravel()),
                        count4=np.array(count), K=np.array(K), ens_agree=np.array(agree, dtype=np.float64),
                        ens_count=np.array(counts, dtype=np.int64), wall_s=np.array(time.time() - t0),
                        threads=np.array(int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))))
    log(f"wrote {path}")
    return path


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--images", type=int, nargs="*", default=None, help="C3 image indices")
    ap.add_argument("--ensemble", type=int, default=0)
    ap.add_argument("--out", default=None, help="write the records here instead of tests/golden/masks "
                                                 "(e.g. gpurun_out/ when the oracle runs on a GPU box's host cores)")
    ap.add_argument("--K", type=int, default=None, help="truncated horizon (record named <cfg>_k<K>.npz)")
    a = ap.parse_args(argv)
    if a.config == "c3":
        for i in (a.images if a.images is not None else [0, 1, 2, 3]):
            compute("c3", i, a.ensemble, out_dir=a.out, K_override=a.K)
    else:
        compute(a.config, None, a.ensemble, out_dir=a.out, K_override=a.K)


if __name__ == "__main__":
    main()
