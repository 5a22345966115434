"""Thin ctypes binding of libsrsb.so (include/srsb.h).  Argument marshalling only: every step
of the Split Bregman SR iteration runs in the library's CUDA kernels.  There is no CPU
fallback: if the library is missing or no GPU is present, construction raises.

Names follow the C ABI: sr_sb_create -> Solver(...), sr_sb_set_image -> Solver.set_image,
sr_sb_iterate -> Solver.iterate, sr_sb_get_phi -> Solver.get_phi.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SRSB_LIB", os.path.join(_HERE, "libsrsb.so"))

SR_OK, SR_ERR_ARG, SR_ERR_SHAPE, SR_ERR_CUDA, SR_ERR_NCCL, SR_ERR_NONFINITE, SR_ERR_STATE, SR_ERR_OOM = \
    0, -1, -2, -3, -4, -5, -6, -7
STATUS_NAMES = {0: "SR_OK", -1: "SR_ERR_ARG", -2: "SR_ERR_SHAPE", -3: "SR_ERR_CUDA", -4: "SR_ERR_NCCL",
                -5: "SR_ERR_NONFINITE", -6: "SR_ERR_STATE", -7: "SR_ERR_OOM"}
NCCL_UNIQUE_ID_BYTES = 128

# every symbol include/srsb.h declares (checked by tests/test_abi.py)
EXPORTS = ["sr_sb_default_params", "sr_sb_create", "sr_sb_set_image", "sr_sb_iterate", "sr_sb_get_phi",
           "sr_sb_get_state", "sr_sb_set_state", "sr_sb_iteration", "sr_sb_sync", "sr_sb_debug_solve",
           "sr_sb_debug_rhs", "sr_sb_debug_wb", "sr_sb_launches_per_iteration", "sr_sb_destroy",
           "sr_sb_last_error", "sr_sb_abi_version", "sr_sb_profile", "sr_sb_create_slab_group",
           "sr_sb_nccl_unique_id", "sr_sb_create_slab_nccl", "sr_sb_local_rows", "sr_sb_set_monitor",
           "sr_sb_get_monitor", "sr_sb_iterate_until", "sr_sb_last_change", "sr_sb_create_dist", "sr_sb_set_iteration",
           "sr_sb_slab_schedule", "sr_sb_a2a_chunks", "sr_sb_tri_constants",
           "sr_sb3_create", "sr_sb3_set_image", "sr_sb3_iterate", "sr_sb3_get_phi", "sr_sb3_get_state",
           "sr_sb3_set_state", "sr_sb3_debug_solve", "sr_sb3_debug_rhs", "sr_sb3_profile", "sr_sb3_sync",
           "sr_sb3_destroy", "sr_sb3_last_error"]
KERNEL_CLASSES = ["rhs", "rows_r2c", "cols_solve", "rows_c2r", "wb", "aos_vert", "aos_horiz",
                  "rhs_r2c", "solve_cluster"]   # sr_kernel_class


class SrsbError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class Params(C.Structure):
    """Mirror of sr_sb_params (include/srsb.h)."""
    _fields_ = [("M", C.c_int), ("N", C.c_int), ("batch", C.c_int),
                ("gamma", C.c_float), ("alpha", C.c_float), ("beta", C.c_float), ("mu", C.c_float),
                ("epsilon", C.c_float), ("l", C.c_float), ("d", C.c_float), ("window", C.c_int),
                ("window_shape", C.c_int), ("tau", C.c_float), ("S", C.c_int), ("rho", C.c_float),
                ("sigma", C.c_float), ("s", C.c_int), ("phi_clip", C.c_float), ("w_proj", C.c_int),
                ("w_mode", C.c_int), ("w_iters", C.c_int), ("b_max", C.c_float), ("phi_solver", C.c_int)]


_lib = None


def lib():
    """Load libsrsb.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -m paper_2003_12693_b200.build`")
        L = C.CDLL(LIB_PATH)
        p, i, st = C.c_void_p, C.c_int, C.c_int
        sig = {
            "sr_sb_default_params": (None, [C.POINTER(Params), i, i, i, i]),
            "sr_sb_create": (st, [C.POINTER(Params), i, p, C.POINTER(p)]),
            "sr_sb_set_image": (st, [p, p, p]),
            "sr_sb_iterate": (st, [p, i]),
            "sr_sb_get_phi": (st, [p, p]),
            "sr_sb_get_state": (st, [p, p, p, p, p]),
            "sr_sb_set_state": (st, [p, p, p, p, p]),
            "sr_sb_iteration": (C.c_longlong, [p]),
            "sr_sb_sync": (st, [p]),
            "sr_sb_debug_solve": (st, [p, p, p]),
            "sr_sb_debug_rhs": (st, [p, p]),
            "sr_sb_debug_wb": (st, [p]),
            "sr_sb_launches_per_iteration": (i, [p]),
            "sr_sb_destroy": (None, [p]),
            "sr_sb_last_error": (C.c_char_p, [p]),
            "sr_sb_abi_version": (i, []),
            "sr_sb_profile": (st, [p, i, C.POINTER(C.c_float), C.POINTER(C.c_int)]),
            "sr_sb_create_slab_group": (st, [C.POINTER(Params), i, p, i, C.POINTER(p)]),
            "sr_sb_nccl_unique_id": (st, [p, i]),
            "sr_sb_create_slab_nccl": (st, [C.POINTER(Params), i, p, i, i, p, C.POINTER(p)]),
            "sr_sb_local_rows": (i, [p]),
            "sr_sb_set_monitor": (st, [p, i]),
            "sr_sb_get_monitor": (st, [p, C.POINTER(C.c_double)]),
            "sr_sb_iterate_until": (st, [p, i, C.c_double, i, C.POINTER(C.c_int)]),
            "sr_sb_last_change": (C.c_double, [p]),
            "sr_sb_create_dist": (st, [C.POINTER(Params), i, p, p, i, i, C.POINTER(p)]),
            "sr_sb_set_iteration": (st, [p, C.c_longlong]),
            "sr_sb_slab_schedule": (i, [i, i, i, i, i, i, i, i, C.POINTER(C.c_longlong), i]),
            "sr_sb_a2a_chunks": (i, [p]),
            "sr_sb_tri_constants": (i, [C.c_float, C.c_float, i, i, i, i, C.POINTER(C.c_double)]),
            "sr_sb3_create": (st, [C.POINTER(Params), i, i, p, C.POINTER(p)]),
            "sr_sb3_set_image": (st, [p, p, p]),
            "sr_sb3_iterate": (st, [p, i]),
            "sr_sb3_get_phi": (st, [p, p]),
            "sr_sb3_get_state": (st, [p, p, p, p, p]),
            "sr_sb3_set_state": (st, [p, p, p, p, p]),
            "sr_sb3_debug_solve": (st, [p, p, p]),
            "sr_sb3_debug_rhs": (st, [p, p]),
            "sr_sb3_profile": (st, [p, i, C.POINTER(C.c_float), C.POINTER(C.c_int)]),
            "sr_sb3_sync": (st, [p]),
            "sr_sb3_destroy": (None, [p]),
            "sr_sb3_last_error": (C.c_char_p, [p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def nccl_unique_id() -> bytes:
    """sr_sb_nccl_unique_id: 128 bytes to broadcast to all ranks before Solver(nccl=...)."""
    buf = C.create_string_buffer(NCCL_UNIQUE_ID_BYTES)
    st = lib().sr_sb_nccl_unique_id(C.cast(buf, C.c_void_p), NCCL_UNIQUE_ID_BYTES)
    if st != SR_OK:
        raise SrsbError(st, lib().sr_sb_last_error(None).decode())
    return buf.raw


def slab_schedule(kind, P, r, Ml, gh, N, k=0, nk=1):
    """sr_sb_slab_schedule: the exchange ops of slab r as a list of (send, peer, buf, off, cnt)."""
    n = lib().sr_sb_slab_schedule(kind, P, r, Ml, gh, N, k, nk, None, 0)
    if n < 0:
        raise SrsbError(SR_ERR_ARG, "bad slab schedule arguments")
    buf = (C.c_longlong * (5 * max(n, 1)))()
    lib().sr_sb_slab_schedule(kind, P, r, Ml, gh, N, k, nk, buf, n)
    return [tuple(int(buf[5 * i + j]) for j in range(5)) for i in range(n)]


def tri_constants(tau, mu, N, k2, L, C_chunks):
    """sr_sb_tri_constants: (r, kappa, rho, closure, mmax) of spectrum column k2 for chunks of L (host logic)."""
    out = (C.c_double * 5)()
    if lib().sr_sb_tri_constants(float(tau), float(mu), int(N), int(k2), int(L), int(C_chunks), out) != 0:
        raise SrsbError(SR_ERR_ARG, "bad tridiagonal-constants arguments")
    return float(out[0]), float(out[1]), float(out[2]), float(out[3]), int(out[4])


def default_params(M, N, batch=1, window=4) -> dict:
    p = Params()
    lib().sr_sb_default_params(C.byref(p), M, N, batch, window)
    return {name: getattr(p, name) for name, _ in Params._fields_}


def _ptr(x):
    """Raw pointer of a contiguous float32 torch tensor (device or host) or numpy array (host)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        if x.dtype != np.float32 or not x.flags["C_CONTIGUOUS"]:
            raise ValueError("numpy arrays must be C-contiguous float32")
        return x.ctypes.data
    import torch
    if isinstance(x, torch.Tensor):
        if x.dtype != torch.float32 or not x.is_contiguous():
            raise ValueError("tensors must be contiguous float32")
        return x.data_ptr()
    raise TypeError(f"unsupported buffer type {type(x)}")


class Solver:
    """One sr_sb context: `batch` images of M x N on one device, bound to one CUDA stream.

    params: any field of sr_sb_params (paper notation); unspecified fields take the
    library defaults (sr_sb_default_params: DESIGN.md §2).
    """

    def __init__(self, M, N, batch=1, window=4, device=None, stream=None, slabs=None, nccl=None, **params):
        """slabs=P: sr_sb_create_slab_group (P row slabs in this process, full-image buffers).
        nccl=(nranks, rank, id_bytes): sr_sb_create_slab_nccl (this rank's slab, local-row buffers)."""
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("srsb needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        p = Params()
        lib().sr_sb_default_params(C.byref(p), M, N, batch, window)   # d = window (reading Q2)
        for k, v in params.items():
            if not hasattr(p, k):
                raise KeyError(f"unknown parameter {k}")
            setattr(p, k, v)
        self.params = {name: getattr(p, name) for name, _ in Params._fields_}
        self.M, self.N, self.batch = M, N, batch
        ctx = C.c_void_p()
        sp = C.c_void_p(stream.cuda_stream)
        if slabs is not None:
            st = lib().sr_sb_create_slab_group(C.byref(p), self.device.index, sp, int(slabs), C.byref(ctx))
        elif nccl is not None:
            nranks, rank, ident = nccl
            buf = C.create_string_buffer(bytes(ident), NCCL_UNIQUE_ID_BYTES)
            st = lib().sr_sb_create_slab_nccl(C.byref(p), self.device.index, sp, int(nranks), int(rank),
                                              C.cast(buf, C.c_void_p), C.byref(ctx))
        else:
            st = lib().sr_sb_create(C.byref(p), self.device.index, sp, C.byref(ctx))
        if st != SR_OK:
            raise SrsbError(st, lib().sr_sb_last_error(None).decode())
        self._ctx = ctx
        self.M_local = int(lib().sr_sb_local_rows(ctx))

    # -- plumbing
    def _check(self, st):
        if st != SR_OK:
            raise SrsbError(st, lib().sr_sb_last_error(self._ctx).decode())

    def _field(self, nch=1):
        import torch
        M = self.M_local
        return torch.empty((self.batch, nch, M, self.N) if nch > 1 else (self.batch, M, self.N),
                           dtype=torch.float32, device=self.device)

    def close(self):
        if getattr(self, "_ctx", None):
            lib().sr_sb_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- the four calls of the boundary
    def set_image(self, image, phi0):
        self._check(lib().sr_sb_set_image(self._ctx, _ptr(image), _ptr(phi0)))

    def iterate(self, K):
        self._check(lib().sr_sb_iterate(self._ctx, int(K)))

    def get_phi(self, out=None):
        out = self._field() if out is None else out
        self._check(lib().sr_sb_get_phi(self._ctx, _ptr(out)))
        return out

    # -- extensions
    def get_state(self, fields=("phi", "w", "b", "g")):
        out = {k: self._field(2 if k in ("w", "b") else 1) for k in fields}
        self._check(lib().sr_sb_get_state(self._ctx, *[_ptr(out.get(k)) for k in ("phi", "w", "b", "g")]))
        return out

    def set_state(self, phi, w, b, g=None):
        self._check(lib().sr_sb_set_state(self._ctx, _ptr(phi), _ptr(w), _ptr(b), _ptr(g)))

    def sync(self):
        self._check(lib().sr_sb_sync(self._ctx))

    @property
    def iteration(self):
        return int(lib().sr_sb_iteration(self._ctx))

    @iteration.setter
    def iteration(self, k):
        self._check(lib().sr_sb_set_iteration(self._ctx, int(k)))

    @property
    def launches_per_iteration(self):
        return int(lib().sr_sb_launches_per_iteration(self._ctx))

    @property
    def a2a_chunks(self):
        """Slab mode: spectrum all-to-all chunks pipelined with the column solve (1 = unchunked)."""
        return int(lib().sr_sb_a2a_chunks(self._ctx))

    def profile(self, K):
        """sr_sb_profile: per kernel class {name: (ms_total, launches)} over K ungraphed iterations."""
        ms = (C.c_float * len(KERNEL_CLASSES))()
        n = (C.c_int * len(KERNEL_CLASSES))()
        self._check(lib().sr_sb_profile(self._ctx, int(K), ms, n))
        return {name: (float(ms[i]), int(n[i])) for i, name in enumerate(KERNEL_CLASSES) if n[i]}

    def set_monitor(self, enable=True):
        self._check(lib().sr_sb_set_monitor(self._ctx, int(bool(enable))))

    def monitor(self):
        """Per image: dict(E_g, E_a, E_r, E_pen, E_total, sweep_change=[..S]) of the last iteration."""
        S = self.params["S"]
        buf = (C.c_double * ((4 + 2 * S) * self.batch))()
        self._check(lib().sr_sb_get_monitor(self._ctx, buf))
        out = []
        p = self.params
        for k in range(self.batch):
            x = buf[k * (4 + 2 * S):(k + 1) * (4 + 2 * S)]
            ch = [(x[4 + 2 * s] ** 0.5) / ((x[5 + 2 * s] ** 0.5) + 1e-6) for s in range(S)]
            out.append(dict(E_g=x[0], E_a=x[1], E_r=x[2], E_pen=x[3],
                            E_total=p["gamma"] * x[0] + p["alpha"] * x[1] + p["beta"] * x[2] + x[3],
                            sweep_change=ch, raw=list(x)))
        return out

    def iterate_until(self, K_max, tol, every=10):
        """sr_sb_iterate_until: returns (iterations run, last relative phi change)."""
        k = C.c_int(0)
        self._check(lib().sr_sb_iterate_until(self._ctx, int(K_max), float(tol), int(every), C.byref(k)))
        return k.value, float(lib().sr_sb_last_change(self._ctx))

    def debug_solve(self, F):
        out = self._field()
        self._check(lib().sr_sb_debug_solve(self._ctx, _ptr(F), _ptr(out)))
        return out

    def debug_rhs(self):
        out = self._field()
        self._check(lib().sr_sb_debug_rhs(self._ctx, _ptr(out)))
        return out

    def debug_wb(self):
        self._check(lib().sr_sb_debug_wb(self._ctx))


class DistSolver(Solver):
    """One rank of an NCCL slab decomposition of ONE image (SURVEY §8(b) srsb.DistSolver): the unique id
    comes from rank 0 through torch.distributed (dist.broadcast_unique_id), then sr_sb_create_dist.
    Buffers hold this rank's rows [1][M/P][N]."""

    def __init__(self, M, N, window=4, device=None, stream=None, group=None, **params):
        import torch
        import torch.distributed as tdist
        from .dist import broadcast_unique_id
        world, rank = tdist.get_world_size(group), tdist.get_rank(group)
        # NCCL broadcasts device tensors only: resolve the device before the id exchange (gloo: CPU)
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        bdev = dev if tdist.get_backend(group) == "nccl" else None
        ident = broadcast_unique_id(nccl_unique_id if rank == 0 else None, group=group, device=bdev)
        super().__init__(M, N, 1, window=window, device=device, stream=stream, nccl=(world, rank, ident), **params)


class Solver3:
    """One sr_sb3 context (NEXT-3): a D x M x N volume on one device, bound to one CUDA stream.
    Fields: phi / volume / g [D][M][N]; w, b [3][D][M][N] (components along i, j, z)."""

    def __init__(self, D, M, N, window=3, device=None, stream=None, **params):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("srsb needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        p = Params()
        lib().sr_sb_default_params(C.byref(p), M, N, 1, window)
        for k, v in params.items():
            if not hasattr(p, k):
                raise KeyError(f"unknown parameter {k}")
            setattr(p, k, v)
        self.params = {name: getattr(p, name) for name, _ in Params._fields_}
        self.D, self.M, self.N = D, M, N
        ctx = C.c_void_p()
        st = lib().sr_sb3_create(C.byref(p), int(D), self.device.index, C.c_void_p(stream.cuda_stream), C.byref(ctx))
        if st != SR_OK:
            raise SrsbError(st, lib().sr_sb3_last_error(None).decode())
        self._ctx = ctx

    def _check(self, st):
        if st != SR_OK:
            raise SrsbError(st, lib().sr_sb3_last_error(self._ctx).decode())

    def _field(self, nch=1):
        import torch
        shape = (nch, self.D, self.M, self.N) if nch > 1 else (self.D, self.M, self.N)
        return torch.empty(shape, dtype=torch.float32, device=self.device)

    def close(self):
        if getattr(self, "_ctx", None):
            lib().sr_sb3_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def set_image(self, volume, phi0):
        self._check(lib().sr_sb3_set_image(self._ctx, _ptr(volume), _ptr(phi0)))

    def iterate(self, K):
        self._check(lib().sr_sb3_iterate(self._ctx, int(K)))

    def get_phi(self, out=None):
        out = self._field() if out is None else out
        self._check(lib().sr_sb3_get_phi(self._ctx, _ptr(out)))
        return out

    def get_state(self):
        out = {"phi": self._field(), "w": self._field(3), "b": self._field(3), "g": self._field()}
        self._check(lib().sr_sb3_get_state(self._ctx, *[_ptr(out[k]) for k in ("phi", "w", "b", "g")]))
        return out

    def set_state(self, phi, w, b, g):
        self._check(lib().sr_sb3_set_state(self._ctx, _ptr(phi), _ptr(w), _ptr(b), _ptr(g)))

    def debug_solve(self, F):
        out = self._field()
        self._check(lib().sr_sb3_debug_solve(self._ctx, _ptr(F), _ptr(out)))
        return out

    def debug_rhs(self):
        out = self._field()
        self._check(lib().sr_sb3_debug_rhs(self._ctx, _ptr(out)))
        return out

    def profile(self, K):
        ms = (C.c_float * len(KERNEL_CLASSES))()
        n = (C.c_int * len(KERNEL_CLASSES))()
        self._check(lib().sr_sb3_profile(self._ctx, int(K), ms, n))
        return {name: (float(ms[i]), int(n[i])) for i, name in enumerate(KERNEL_CLASSES) if n[i]}

    def sync(self):
        self._check(lib().sr_sb3_sync(self._ctx))
