#!/usr/bin/env python
"""Benchmark of the Split Bregman SR iteration on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU, NCCL)

Workload: BASELINE configs[2] = C3, a batch of 64 independent 1024x1024 fp32
images, 1000 Split Bregman iterations each, window radius 4 -- the config the metric's
"1/2/4/8 B200" batch scaling and "% of HBM peak" are quoted on.  One STEP is the whole job
for the batch: set_image (edge indicator Eq. 1 + init, §8(a) rows a0-a1) and 1000 outer
iterations (rows a2-a5: 3 x [RHS Eq. 37 + FFT solve Eq. 33] + w/b update Eq. 41/42/40/23).
With N GPUs the 64 images are sharded by image (no collective in the loop), so total work is
fixed ("strong").  value = 64 * 1024^2 * 1000 * steps / (max over ranks of the device time) / 1e6.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "megapixel-iterations/s per SB-SR iteration"
UNIT = "Mpx-iter/s"
# algorithmic HBM bytes per pixel per launch of each kernel class
BYTES_PER_PX = {"rhs": 28.0, "rows_r2c": 8.0, "cols_solve": 8.0, "rows_c2r": 12.0, "wb": 40.0,
                "aos_vert": 8.0, "aos_horiz": 12.0,   # aos_vert: register-chunk kernel (M <= 2048)
                "rhs_r2c": 28.0,   # fused RHS + row R2C: phi, w1, w2, b1, b2, g in, packed half spectrum out
                "solve_cluster": 12.0}   # small images, one-kernel solve: D and psi in, phi out (the spectrum stays on chip)
MODEL_BYTES_PER_PX_ITER = 172.0   # SURVEY.md §8(d) fused model (S = 3)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5", "v3d"],
                    help="v3d: the 3-D extension (NEXT-3) on a synthetic 128^3 volume")
    ap.add_argument("--images", type=int, default=None, help="override the batch (C3 only)")
    ap.add_argument("--iters", type=int, default=None, help="override iterations per step")
    ap.add_argument("--phi-solver", default="fft", choices=["fft", "aos"],
                    help="phi sub-problem: FFT solve Eq. (31)-(33) (north star) or the AOS variant (P:427)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-fft-ref", action="store_true", help="skip the cuFFT reference timing (SURVEY §8(d))")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def workload(args):
    from synth import CONFIGS
    cfg = dict(CONFIGS[args.config])
    if args.images:
        cfg["batch"] = args.images
    if args.iters:
        cfg["K"] = args.iters
    cfg["phi_solver"] = {"fft": 0, "aos": 1}[args.phi_solver]
    return cfg


class ClockSampler:
    """nvidia-smi equivalent via NVML, sampled during the timed region (B200_PROFILING.md clocks line)."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self._stop = threading.Event()
        self.ok = True
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.ok = False

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.1)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_model() -> str:
    """The host CPU's model name (/proc/cpuinfo), for the cpu_baseline record."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline_oracle(cfg, target_s=20.0):
    """The float64 oracle as it stands, on this host's cores, on a bounded sample of the workload:
    for C3 four images spread over the batch (0, 21, 42, 63), for the single-image configs the image;
    the same number of iterations on each, as many as fit ~target_s in total (at least 1)."""
    import numpy as np
    import oracle
    from synth import make_config
    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    imgs = [0, 21, 42, 63] if cfg["name"] == "c3" else [None]
    c = make_config(cfg["name"], images=imgs) if cfg["name"] == "c3" else make_config(cfg["name"])
    p = dict(c["params"], phi_solver=cfg["phi_solver"])
    M, N = c["image"].shape[1:]
    states = []
    for b in range(len(imgs)):
        g = oracle.edge(c["image"][b], p["sigma"], p["rho"], p["s"])
        states.append((oracle.init(c["phi0"][b]), g))
    t0 = time.perf_counter()
    oracle.iterate(p, states[0][0], states[0][1], 1)
    t1 = time.perf_counter() - t0
    k = max(1, int(target_s / len(imgs) / max(t1, 1e-3)))
    t0 = time.perf_counter()
    for b, (st, g) in enumerate(states):
        oracle.iterate(p, st, g, k - 1 if b == 0 else k)
    t = time.perf_counter() - t0 + t1
    del np
    return {"value": len(imgs) * M * N * k / t / 1e6, "unit": UNIT, "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(),
            "sample": f"{len(imgs)} image(s) of {cfg['name']} ({M}x{N}"
                      f"{', images ' + str(imgs) if imgs[0] is not None else ''}), {k} SB iterations each, "
                      f"float64 C oracle, OMP_NUM_THREADS={os.environ.get('OMP_NUM_THREADS')}, {t:.1f} s"}


def cufft_reference(nb, M, N, dev, stream, kernels, reps=5, solver_factory=None):
    """cuFFT R2C + C2R (torch.fft, i.e. cuFFT) on the same batch of M x N fp32 fields,
    timed next to our three-pass solve (k_rows_r2c + k_cols_solve + k_rows_c2r, which also applies
    the symbol and the increment).  Never on the hot path; measured after the timed regions.  When the
    measured context fuses the row R2C into the RHS kernel, the three passes are profiled on a second,
    unfused context (SRSB_FUSE=0) of the same shape (solver_factory)."""
    import torch
    if "rows_r2c" not in kernels and solver_factory is not None:
        os.environ["SRSB_FUSE"] = "0"
        try:
            sv2, img, phi0 = solver_factory()
            sv2.set_image(img, phi0)
            prof = sv2.profile(1)
            sv2.sync()
            sv2.close()
        finally:
            del os.environ["SRSB_FUSE"]
        kernels = {k: {"ms_per_launch": v[0] / v[1]} for k, v in prof.items()}
    x = torch.randn(nb, M, N, device=dev, dtype=torch.float32)
    with torch.cuda.stream(stream):
        for _ in range(2):
            y = torch.fft.irfft2(torch.fft.rfft2(x), s=(M, N))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            y = torch.fft.irfft2(torch.fft.rfft2(x), s=(M, N))
        e1.record(stream)
        torch.cuda.synchronize()
    cufft_ms = e0.elapsed_time(e1) / reps
    ours = sum(kernels[k]["ms_per_launch"] for k in ("rows_r2c", "cols_solve", "rows_c2r") if k in kernels)
    del x, y
    return {"cufft_rfft2_irfft2_ms": cufft_ms, "ours_r2c_cols_c2r_ms": ours if ours else None,
            "batch": nb, "M": M, "N": N,
            "note": "ours includes the symbol division and the increment/clamp epilogue; cuFFT is transforms only"}


def run_reference(args, cfg, rank):
    """--impl reference: the float64 CPU oracle, rank 0 only."""
    if rank != 0:
        return None
    import oracle
    from synth import make_config
    oracle.build()
    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    c = make_config(cfg["name"], images=[0]) if cfg["name"] == "c3" else make_config(cfg["name"])
    p = dict(c["params"], phi_solver=cfg["phi_solver"])
    img, phi0 = c["image"][0], c["phi0"][0]
    M, N = img.shape
    g = oracle.edge(img, p["sigma"], p["rho"], p["s"])
    st = oracle.init(phi0)
    # each step: one outer iteration of one image (bounded sample of the workload)
    for _ in range(args.warmup):
        oracle.iterate(p, st, g, 1)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.iterate(p, st, g, 1)
    t = time.perf_counter() - t0
    value = M * N * args.steps / t / 1e6
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_json(cfg, args.gpus),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
                             "sample": f"each step = 1 SB iteration of image 0 of {cfg['name']} ({M}x{N}), "
                                       f"float64 C oracle, OMP_NUM_THREADS={os.environ['OMP_NUM_THREADS']}"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def config_json(cfg, ngpu):
    return {"workload": f"{cfg['name']}: {cfg['batch']} x {cfg['M']}x{cfg['N']} fp32 images, {cfg['K']} SB "
                        f"iterations each, window radius {cfg['window']}, S=3",
            "config_index": cfg["index"], "images": cfg["batch"], "M": cfg["M"], "N": cfg["N"],
            "iterations_per_step": cfg["K"], "window": cfg["window"], "S": 3,
            "phi_solver": ["fft (Eq. 31-33)", "aos (P:427)"][cfg["phi_solver"]],
            "parallelism": {"c3": f"batch-shard x{ngpu} (images split across GPUs, no collective in the loop)",
                            "c5": (f"slab x{ngpu} (row slabs; NCCL halo send/recv + all-to-all spectrum transpose)"
                                   if ngpu > 1 else "single GPU, whole image")}.get(
                cfg["name"], f"replicas x{ngpu} (independent copies of the one-image config)" if ngpu > 1
                else "single GPU"),
            "l2": "inputs larger than L2 (44 B/px of state per GPU)" if cfg["name"] != "c1" and cfg["name"] != "c2"
                  else "L2-resident config (state < 126 MB): latency-bound, not an HBM measurement"}


VOL_BYTES_PER_VOX = {"rhs": 36.0, "rows_r2c": 8.0, "cols_solve": 8.0, "rows_c2r": 12.0, "wb": 56.0}


def run_volume(args, world, rank, local):
    """--config v3d: the 3-D extension on a synthetic 128^3 volume (synth.volumes),
    R = 3, K = 200 iterations per step; value in Mvox-iter/s.  N > 1: independent replicas."""
    import numpy as np
    import torch
    from paper_2003_12693_b200 import Solver3
    from synth import make_volume
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    from paper_2003_12693_b200.dist import max_over_ranks as _max_over_ranks
    shape, R = (128, 128, 128), 3
    K = args.iters or 200
    v = make_volume(shape, n=12, window=R, seed=0)
    p = v["params"]
    keys = ("gamma", "alpha", "beta", "mu", "epsilon", "l", "d", "window_shape", "tau", "S", "rho", "sigma", "s",
            "phi_clip", "w_proj", "w_mode", "w_iters")
    stream = torch.cuda.Stream(dev)
    sv = Solver3(*shape, window=R, device=local, stream=stream, **{k: p[k] for k in keys})
    vol_d = torch.from_numpy(v["volume"]).to(dev)
    phi_d = torch.from_numpy(v["phi0"]).to(dev)
    out_d = torch.empty_like(phi_d)
    nvox = int(np.prod(shape))

    def step():
        sv.set_image(vol_d, phi_d)
        sv.iterate(K)
        sv.get_phi(out_d)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            e0.record(stream)
            for _ in range(args.steps):
                step()
            e1.record(stream)
            torch.cuda.synchronize()
    sv.sync()
    ms = _max_over_ranks(e0.elapsed_time(e1), device=dev)
    value = world * nvox * K * args.steps / (ms / 1e3) / 1e6
    peak, peak_src = peaks()
    sv.set_image(vol_d, phi_d)
    prof = sv.profile(2)
    dom = max(prof, key=lambda k: prof[k][0])
    kern = {k: {"ms_per_launch": a / n, "launches_per_iter": n // 2,
                "GBs": VOL_BYTES_PER_VOX[k] * nvox / (a / n / 1e3) / 1e9} for k, (a, n) in prof.items()}
    roof = {"bound": "hbm", "kernel": dom, "achieved": kern[dom]["GBs"], "peak": peak, "unit": "GB/s",
            "frac": kern[dom]["GBs"] / peak, "traffic": None, "peak_source": peak_src,
            "bytes_per_vox_per_launch": VOL_BYTES_PER_VOX[dom], "kernels": kern}
    if rank == 0:
        print(json.dumps({"metric": "megavoxel-iterations/s per SB-SR iteration (3-D extension, NEXT-3)",
                          "value": value, "unit": "Mvox-iter/s", "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                          "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                          "config": {"workload": f"v3d: one {shape[0]}x{shape[1]}x{shape[2]} fp32 volume (12 random "
                                                 f"ellipsoids, noise 0.15), {K} SB iterations, ball radius {R}, S=3",
                                     "l2": "state 46 B/voxel x 2 Mvox = 96 MB: partly L2-resident",
                                     "parallelism": f"replicas x{world}" if world > 1 else "single GPU"},
                          # per iteration: S x (rhs, r2c, solve, c2r) + wb; the lines solve (D >= 16, M >= 32) is 5 kernels
                          # (line FFT, unpack, z solve, repack, inverse line FFT), the plane solve 1
                          "roofline": roof,
                          "gpu_launches": args.steps * (5 + K * (3 * (3 + (5 if shape[0] >= 16 and shape[1] >= 32 and
                                                                          os.environ.get("SRSB_VOL_SOLVE", "")[:1] != "p"
                                                                          else 1)) + 1)) * world,
                          "clocks": clk.summary()}), flush=True)
    sv.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def run_reference_volume(args, rank):
    """--impl reference --config v3d: the 3-D float64 oracle on a 64^3 crop of the v3d recipe (bounded
    sample), one SB iteration per step, rank 0 only."""
    if rank != 0:
        return None
    import oracle
    from synth import make_volume
    oracle.build()
    cores = len(os.sched_getaffinity(0))
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    v = make_volume((64, 64, 64), n=4, window=3, seed=0)
    p = v["params"]
    g = oracle.edge3(v["volume"], p["sigma"], p["rho"], p["s"])
    st = oracle.init3(v["phi0"])
    for _ in range(args.warmup):
        oracle.iterate3(p, st, g, 1)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.iterate3(p, st, g, 1)
    t = time.perf_counter() - t0
    value = 64 ** 3 * args.steps / t / 1e6
    return {"impl": "reference", "metric": "megavoxel-iterations/s per SB-SR iteration (3-D extension, NEXT-3)",
            "value": value, "unit": "Mvox-iter/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": "v3d recipe, 64^3 crop, 1 SB iteration per step, ball radius 3, S=3"},
            "cpu_baseline": {"value": value, "unit": "Mvox-iter/s", "cores": cores, "kind": "oracle",
                             "sample": f"64^3 volume, 1 SB iteration per step, float64 C oracle, "
                                       f"OMP_NUM_THREADS={os.environ['OMP_NUM_THREADS']}"},
            "e2e": {"value": value, "unit": "Mvox-iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    if args.config == "v3d" and args.impl == "reference":
        out = run_reference_volume(args, int(os.environ.get("RANK", "0")))
        if out is not None:
            print(json.dumps(out), flush=True)
        return 0
    if args.config == "v3d" and args.impl != "reference":
        return run_volume(args, int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
                          int(os.environ.get("LOCAL_RANK", "0")))
    cfg = workload(args)
    cfg["name"] = args.config
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        out = run_reference(args, cfg, rank)
        if out is not None:
            print(json.dumps(out), flush=True)
        return 0

    import numpy as np
    import torch
    from paper_2003_12693_b200 import Solver
    from synth import make_config

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    B = cfg["batch"]
    from paper_2003_12693_b200.dist import max_over_ranks as _max_over_ranks, shard
    # work split: C3 shards images across ranks; C5 splits its one image into row
    # slabs (NCCL halos + all-to-all transpose); C1/C2/C4 run as independent replicas
    if args.config == "c3":
        mode = "batch-shard"
    elif args.config == "c5" and world > 1:
        mode = "slab"
    else:
        mode = "replica" if world > 1 else "single"
    if mode == "slab" and cfg["phi_solver"]:
        raise SystemExit("--phi-solver aos is for whole-image contexts (slab mode uses the FFT solve)")
    M, N, K = cfg["M"], cfg["N"], cfg["K"]
    if mode == "batch-shard":
        s0, s1 = shard(B, world, rank)
        data = make_config("c3", images=range(s0, s1))
        nb = s1 - s0
    else:
        data = make_config(args.config)
        nb = 1
    p = data["params"]
    keys = ("gamma", "alpha", "beta", "mu", "epsilon", "l", "d", "window_shape", "tau", "S", "rho", "sigma",
            "s", "phi_clip", "w_proj", "w_mode", "w_iters")
    stream = torch.cuda.Stream(dev)
    extra = {}
    if mode == "slab":
        from paper_2003_12693_b200.dist import broadcast_unique_id
        from paper_2003_12693_b200.srsb import nccl_unique_id
        ident = broadcast_unique_id(nccl_unique_id if rank == 0 else None, device=dev)
        extra = dict(nccl=(world, rank, ident))
        rows = slice(rank * M // world, (rank + 1) * M // world)
        data["image"] = np.ascontiguousarray(data["image"][:, rows])
        data["phi0"] = np.ascontiguousarray(data["phi0"][:, rows])
    sv = Solver(M, N, nb, window=p["window"], device=local, stream=stream, phi_solver=cfg["phi_solver"],
                **{k: p[k] for k in keys}, **extra)
    img_d = torch.from_numpy(data["image"]).to(dev)
    phi0_d = torch.from_numpy(data["phi0"]).to(dev)
    out_d = torch.empty_like(phi0_d)
    torch.cuda.synchronize()

    def step_device():
        sv.set_image(img_d, phi0_d)
        sv.iterate(K)
        sv.get_phi(out_d)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x):
        return _max_over_ranks(x, device=dev)

    # ---------------------------------------------------------------- device-resident timing (value)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step_device()
        sv.sync()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            e0.record(stream)
            for _ in range(args.steps):
                step_device()
            e1.record(stream)
            torch.cuda.synchronize()
        sv.sync()
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1))
    ms_step = ms / args.steps
    px_total = {"batch-shard": B * M * N, "slab": M * N, "replica": world * M * N, "single": M * N}[mode]
    value = px_total * K * args.steps / (ms / 1e3) / 1e6

    # ---------------------------------------------------------------- per-kernel roofline (profile pass)
    peak, peak_src = peaks()
    px_rank = nb * (M // world if mode == "slab" else M) * N
    step_model = {"bytes_per_px_iter": MODEL_BYTES_PER_PX_ITER,
                  "achieved_GBs": MODEL_BYTES_PER_PX_ITER * px_rank * K / (ms_step / 1e3) / 1e9}
    step_model["frac"] = step_model["achieved_GBs"] / peak
    if mode != "slab":
        sv.set_image(img_d, phi0_d)
        prof_iters = 2
        prof = sv.profile(prof_iters)
        dom = max(prof, key=lambda k: prof[k][0])
        dom_ms, dom_n = prof[dom]
        achieved = BYTES_PER_PX[dom] * px_rank / (dom_ms / dom_n / 1e3) / 1e9
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tpath):
            t = json.load(open(tpath))
            if t.get("workload") == args.config and dom in t.get("per_launch_bytes", {}):
                traffic = t["per_launch_bytes"][dom]
        iter_ms = sum(v[0] for v in prof.values()) / prof_iters
        kernels = {k: {"ms_per_launch": v[0] / v[1], "launches_per_iter": v[1] // prof_iters,
                       "share": v[0] / sum(x[0] for x in prof.values()),
                       "GBs": BYTES_PER_PX[k] * px_rank / (v[0] / v[1] / 1e3) / 1e9} for k, v in prof.items()}
        roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                    "frac": achieved / peak, "frac_vs_datasheet_8TBs": achieved / 8000.0,
                    "traffic": traffic, "peak_source": peak_src,
                    "bytes_per_px_per_launch": BYTES_PER_PX[dom], "step_model": step_model,
                    "kernels": kernels, "profiled_iteration_ms": iter_ms}
    else:   # slab mode: no per-kernel profile entry; the whole-step model per rank
        roofline = {"bound": "hbm", "kernel": "step (slab: kernels + NCCL halos / all-to-all)",
                    "achieved": step_model["achieved_GBs"], "peak": peak, "unit": "GB/s",
                    "frac": step_model["frac"], "traffic": None, "peak_source": peak_src,
                    "bytes_per_px_per_launch": None, "step_model": step_model}

    # ---------------------------------------------------------------- end to end through host buffers
    e2e = None
    if not args.no_e2e:
        img_h = torch.from_numpy(data["image"]).pin_memory()
        phi0_h = torch.from_numpy(data["phi0"]).pin_memory()
        out_h = torch.empty_like(phi0_h).pin_memory()

        def step_host():
            sv.set_image(img_h, phi0_h)      # H2D inside the call
            sv.iterate(K)
            sv.get_phi(out_h)                # D2H inside the call
        with torch.cuda.stream(stream):
            step_host()
            sv.sync()
            barrier()
            torch.cuda.synchronize()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            for _ in range(args.steps):
                step_host()
            f1.record(stream)
            torch.cuda.synchronize()
            sv.sync()
        barrier()
        ems = max_over_ranks(f0.elapsed_time(f1))
        e2e = {"value": px_total * K * args.steps / (ems / 1e3) / 1e6, "unit": UNIT,
               "h2d_bytes_per_step": int(img_h.numel() * 4 + phi0_h.numel() * 4) * world,
               "d2h_bytes_per_step": int(out_h.numel() * 4) * world, "ms_per_step": ems / args.steps}

    launches = args.steps * (4 + K * sv.launches_per_iteration)
    fft_ref = None
    if rank == 0 and mode != "slab" and not args.no_fft_ref and "kernels" in roofline:
        def factory():
            return (Solver(M, N, nb, window=p["window"], device=local, stream=stream, phi_solver=cfg["phi_solver"],
                           **{k: p[k] for k in keys}), img_d, phi0_d)
        fft_ref = cufft_reference(nb, M, N, dev, stream, roofline["kernels"], solver_factory=factory)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline_oracle(cfg)
    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
               "scaling": "weak" if mode == "replica" else "strong",
               "vs_baseline": None, "dtype": "f32", "data": "synthetic", "config": dict(config_json(cfg, world), mode=mode),
               "value_per_gpu": value / world,
               "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches * world,
               "clocks": clk.summary(), "fft_reference": fft_ref}
        print(json.dumps(out), flush=True)
    sv.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
