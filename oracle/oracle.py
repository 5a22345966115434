"""ctypes wrapper around oracle/sr_oracle.c (plain C, float64).

TEST INFRASTRUCTURE ONLY -- see oracle/__init__.py.  Every function converts
its inputs to C-contiguous float64 and calls the C routine of the same name;
there is no arithmetic of the method in this file.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sr_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

__all__ = ["build", "Params", "H", "delta", "delta_prime", "h", "h_prime", "grad", "div", "edge",
           "fft", "fft2", "symbol", "solve", "window_sum", "rhs", "shrink", "project", "wb",
           "init", "sweep", "iterate", "label", "run", "lib", "energy", "thomas_neumann", "solve_aos",
           "grad3", "div3", "edge3", "fft3", "symbol3", "solve3", "window_sum3", "rhs3", "shrink3", "project3",
           "wb3", "init3", "iterate3", "run3"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2 -ffp-contract=off -fopenmp, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
               "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.check_call(cmd)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        d, i, p = C.c_double, C.c_int, C.c_void_p
        sig = {
            "orc_H": (d, [d, d]), "orc_delta": (d, [d, d]), "orc_delta_prime": (d, [d, d]),
            "orc_h": (d, [d, d, d]), "orc_h_prime": (d, [d, d, d]),
            "orc_grad": (None, [i, i, p, p, p]), "orc_div": (None, [i, i, p, p, p]),
            "orc_edge": (None, [i, i, p, d, d, i, p]),
            "orc_fft": (i, [i, p, p, i]), "orc_fft2": (i, [i, i, p, p, i]),
            "orc_symbol": (d, [i, i, d, d, i, i]), "orc_solve": (i, [i, i, d, d, p, p]),
            "orc_window_sum": (None, [i, i, i, d, i, p, p, p, p]),
            "orc_rhs": (None, [i, i, p, p, p, p, p, p, p, p]),
            "orc_shrink": (None, [d, d, d, p, p]), "orc_project": (None, [i, d, d, p, p]),
            "orc_wb": (None, [i, i, p, p, p, p, p, p, p]),
            "orc_init": (None, [i, i, p, p, p, p, p, p]),
            "orc_sweep": (i, [i, i, p, p, p, p, p, p, p]),
            "orc_iterate": (i, [i, i, p, p, p, p, p, p, p, i]),
            "orc_label": (i, [i, i, p, i, p]),
            "orc_energy": (None, [i, i, p, p, p, p, p, p, p, p]),
            "orc_thomas_neumann": (None, [i, d, p, p]),
            "orc_solve_aos": (None, [i, i, d, d, p, p]),
            "orc3_grad": (None, [i, i, i, p, p, p, p]), "orc3_div": (None, [i, i, i, p, p, p, p]),
            "orc3_edge": (None, [i, i, i, p, d, d, i, p]), "orc3_fft3": (i, [i, i, i, p, p, i]),
            "orc3_symbol": (d, [i, i, i, d, d, i, i, i]), "orc3_solve": (i, [i, i, i, d, d, p, p]),
            "orc3_window_sum": (None, [i, i, i, i, d, i, p, p, p, p, p, p]),
            "orc3_rhs": (None, [i, i, i, p] + [p] * 9),
            "orc3_shrink": (None, [p, d, p]), "orc3_project": (None, [i, p, p]),
            "orc3_wb": (None, [i, i, i, p] + [p] * 8),
            "orc3_init": (None, [i, i, i] + [p] * 8),
            "orc3_iterate": (i, [i, i, i, p] + [p] * 8 + [i]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(_lib, name)
            fn.restype = res
            fn.argtypes = args
    return _lib


class Params(C.Structure):
    """Mirror of orc_params in sr_oracle.c."""
    _fields_ = [("gamma", C.c_double), ("alpha", C.c_double), ("beta", C.c_double), ("mu", C.c_double),
                ("epsilon", C.c_double), ("l", C.c_double), ("d", C.c_double), ("window", C.c_int),
                ("window_shape", C.c_int), ("tau", C.c_double), ("S", C.c_int), ("phi_clip", C.c_double),
                ("w_proj", C.c_int), ("w_mode", C.c_int), ("w_iters", C.c_int), ("phi_solver", C.c_int)]

    @classmethod
    def from_dict(cls, p: dict) -> "Params":
        q = cls()
        for name, _ in cls._fields_:
            setattr(q, name, p.get(name, 0) if name == "phi_solver" else p[name])
        return q


def _d(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


def _P(p):
    return C.byref(p if isinstance(p, Params) else Params.from_dict(p))


# pointwise ------------------------------------------------------------
def H(x, eps):
    return float(lib().orc_H(x, eps))


def delta(x, eps):
    return float(lib().orc_delta(x, eps))


def delta_prime(x, eps):
    return float(lib().orc_delta_prime(x, eps))


def h(x, eps, l):
    return float(lib().orc_h(x, eps, l))


def h_prime(x, eps, l):
    return float(lib().orc_h_prime(x, eps, l))


# fields ---------------------------------------------------------------
def grad(phi):
    phi = _d(phi)
    M, N = phi.shape
    g1, g2 = np.empty_like(phi), np.empty_like(phi)
    lib().orc_grad(M, N, _ptr(phi), _ptr(g1), _ptr(g2))
    return g1, g2


def div(u1, u2):
    u1, u2 = _d(u1), _d(u2)
    M, N = u1.shape
    out = np.empty_like(u1)
    lib().orc_div(M, N, _ptr(u1), _ptr(u2), _ptr(out))
    return out


def edge(f, sigma=1.0, rho=1.0, s=2):
    f = _d(f)
    M, N = f.shape
    g = np.empty_like(f)
    lib().orc_edge(M, N, _ptr(f), sigma, rho, s, _ptr(g))
    return g


def fft(x, inverse=False):
    x = np.asarray(x, dtype=np.complex128)
    re, im = _d(x.real.copy()), _d(x.imag.copy())
    if lib().orc_fft(len(x), _ptr(re), _ptr(im), int(inverse)) != 0:
        raise ValueError("length must be a power of two")
    return re + 1j * im


def fft2(x, inverse=False):
    x = np.asarray(x, dtype=np.complex128)
    M, N = x.shape
    re, im = _d(x.real.copy()), _d(x.imag.copy())
    if lib().orc_fft2(M, N, _ptr(re), _ptr(im), int(inverse)) != 0:
        raise ValueError("sizes must be powers of two")
    return re + 1j * im


def symbol(M, N, tau, mu, k1, k2):
    return float(lib().orc_symbol(M, N, tau, mu, k1, k2))


def solve(F, tau, mu, check=True):
    F = _d(F)
    M, N = F.shape
    phi = np.empty_like(F)
    bad = lib().orc_solve(M, N, tau, mu, _ptr(F), _ptr(phi))
    if check and bad:
        raise FloatingPointError("imaginary part of the solve exceeds 1e-12 max|F| (Q11)")
    return phi


def thomas_neumann(f, c):
    """(I - c A) x = f on one line, A the Neumann 1-D second difference (Thomas algorithm)."""
    f = _d(f)
    x = np.empty_like(f)
    lib().orc_thomas_neumann(len(f), c, _ptr(f), _ptr(x))
    return x


def solve_aos(F, tau, mu):
    """AOS phi solve of P:427: 1/2 [(I - 2 tau mu A_1)^-1 + (I - 2 tau mu A_2)^-1] F."""
    F = _d(F)
    M, N = F.shape
    phi = np.empty_like(F)
    lib().orc_solve_aos(M, N, tau, mu, _ptr(F), _ptr(phi))
    return phi


def window_sum(u1, u2, R, d, shape=0):
    u1, u2 = _d(u1), _d(u2)
    M, N = u1.shape
    v1, v2 = np.empty_like(u1), np.empty_like(u1)
    lib().orc_window_sum(M, N, R, d, shape, _ptr(u1), _ptr(u2), _ptr(v1), _ptr(v2))
    return v1, v2


def rhs(p, psi, w1, w2, b1, b2, g):
    psi, w1, w2, b1, b2, g = map(_d, (psi, w1, w2, b1, b2, g))
    M, N = psi.shape
    F = np.empty_like(psi)
    lib().orc_rhs(M, N, _P(p), _ptr(psi), _ptr(w1), _ptr(w2), _ptr(b1), _ptr(b2), _ptr(g), _ptr(F))
    return F


def shrink(B1, B2, t):
    o1, o2 = C.c_double(), C.c_double()
    lib().orc_shrink(B1, B2, t, C.byref(o1), C.byref(o2))
    return o1.value, o2.value


def project(mode, a1, a2):
    o1, o2 = C.c_double(), C.c_double()
    lib().orc_project(mode, a1, a2, C.byref(o1), C.byref(o2))
    return o1.value, o2.value


def wb(p, phi, w1, w2, b1, b2, g):
    """Returns new (w1, w2, b1, b2); inputs are not modified."""
    phi, g = _d(phi), _d(g)
    w1, w2, b1, b2 = (np.array(a, dtype=np.float64, copy=True) for a in (w1, w2, b1, b2))
    M, N = phi.shape
    lib().orc_wb(M, N, _P(p), _ptr(phi), _ptr(w1), _ptr(w2), _ptr(b1), _ptr(b2), _ptr(g))
    return w1, w2, b1, b2


def init(phi0):
    phi0 = _d(phi0)
    M, N = phi0.shape
    out = [np.empty_like(phi0) for _ in range(5)]
    lib().orc_init(M, N, _ptr(phi0), *[_ptr(a) for a in out])
    return dict(phi=out[0], w1=out[1], w2=out[2], b1=out[3], b2=out[4])


def sweep(p, psi, w1, w2, b1, b2, g):
    psi = np.array(psi, dtype=np.float64, copy=True)
    w1, w2, b1, b2, g = map(_d, (w1, w2, b1, b2, g))
    M, N = psi.shape
    bad = lib().orc_sweep(M, N, _P(p), _ptr(psi), _ptr(w1), _ptr(w2), _ptr(b1), _ptr(b2), _ptr(g))
    if bad:
        raise FloatingPointError("imaginary part of the solve exceeds tolerance (Q11)")
    return psi


def iterate(p, state, g, K):
    """Advance `state` (dict phi, w1, w2, b1, b2 of float64 arrays) by K outer iterations, in place."""
    g = _d(g)
    for k in ("phi", "w1", "w2", "b1", "b2"):
        state[k] = np.array(state[k], dtype=np.float64, copy=True, order="C")
    M, N = g.shape
    bad = lib().orc_iterate(M, N, _P(p), *[_ptr(state[k]) for k in ("phi", "w1", "w2", "b1", "b2")], _ptr(g), K)
    if bad:
        raise FloatingPointError(f"{bad} solves failed the imaginary-part check (Q11)")
    return state


def energy(p, phi, w1, w2, b1, b2, g):
    """(E_g, E_a, E_r, E_pen) of Eq. (22) at (phi, w, b); total = gamma E_g + alpha E_a + beta E_r + E_pen."""
    phi, w1, w2, b1, b2, g = map(_d, (phi, w1, w2, b1, b2, g))
    M, N = phi.shape
    out = np.zeros(4)
    lib().orc_energy(M, N, _P(p), _ptr(phi), _ptr(w1), _ptr(w2), _ptr(b1), _ptr(b2), _ptr(g), _ptr(out))
    return tuple(out)


def label(mask, conn=4):
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    M, N = m.shape
    lab = np.empty((M, N), dtype=np.int32)
    n = lib().orc_label(M, N, _ptr(m), conn, _ptr(lab))
    return int(n), lab


def run(p, image, phi0, K):
    """Algorithm 1 from scratch for one image: g (Eq. 1), init, K iterations."""
    g = edge(image, p["sigma"], p["rho"], p["s"])
    st = init(phi0)
    iterate(p, st, g, K)
    st["g"] = g
    return st


# 3-D extension (NEXT-3, reading Q26) --------------------------------------------------------------
# Volumes are [D][M][N]; vector fields are tuples (c1, c2, c3) = (along rows i, columns j, depth z).
def grad3(phi):
    phi = _d(phi)
    D, M, N = phi.shape
    g = [np.empty_like(phi) for _ in range(3)]
    lib().orc3_grad(D, M, N, _ptr(phi), *[_ptr(a) for a in g])
    return tuple(g)


def div3(u1, u2, u3):
    u1, u2, u3 = _d(u1), _d(u2), _d(u3)
    D, M, N = u1.shape
    out = np.empty_like(u1)
    lib().orc3_div(D, M, N, _ptr(u1), _ptr(u2), _ptr(u3), _ptr(out))
    return out


def edge3(f, sigma=1.0, rho=1.0, s=2):
    f = _d(f)
    D, M, N = f.shape
    g = np.empty_like(f)
    lib().orc3_edge(D, M, N, _ptr(f), sigma, rho, s, _ptr(g))
    return g


def fft3(x, inverse=False):
    x = np.asarray(x, dtype=np.complex128)
    D, M, N = x.shape
    re, im = _d(x.real.copy()), _d(x.imag.copy())
    if lib().orc3_fft3(D, M, N, _ptr(re), _ptr(im), int(inverse)) != 0:
        raise ValueError("sizes must be powers of two")
    return re + 1j * im


def symbol3(D, M, N, tau, mu, k3, k1, k2):
    return float(lib().orc3_symbol(D, M, N, tau, mu, k3, k1, k2))


def solve3(F, tau, mu, check=True):
    F = _d(F)
    D, M, N = F.shape
    phi = np.empty_like(F)
    bad = lib().orc3_solve(D, M, N, tau, mu, _ptr(F), _ptr(phi))
    if check and bad:
        raise FloatingPointError("imaginary part of the 3-D solve exceeds 1e-12 max|F| (Q11)")
    return phi


def window_sum3(u1, u2, u3, R, d, shape=0):
    u1, u2, u3 = _d(u1), _d(u2), _d(u3)
    D, M, N = u1.shape
    v = [np.empty_like(u1) for _ in range(3)]
    lib().orc3_window_sum(D, M, N, R, d, shape, _ptr(u1), _ptr(u2), _ptr(u3), *[_ptr(a) for a in v])
    return tuple(v)


def rhs3(p, psi, w, b, g):
    """w, b: 3-tuples of [D][M][N] arrays."""
    psi, g = _d(psi), _d(g)
    w = [_d(a) for a in w]
    b = [_d(a) for a in b]
    D, M, N = psi.shape
    F = np.empty_like(psi)
    lib().orc3_rhs(D, M, N, _P(p), _ptr(psi), *[_ptr(a) for a in w], *[_ptr(a) for a in b], _ptr(g), _ptr(F))
    return F


def shrink3(B, t):
    B = _d(B)
    o = np.empty(3)
    lib().orc3_shrink(_ptr(B), t, _ptr(o))
    return o


def project3(mode, a):
    a = _d(a)
    o = np.empty(3)
    lib().orc3_project(mode, _ptr(a), _ptr(o))
    return o


def wb3(p, phi, w, b, g):
    """Returns new (w, b) 3-tuples; inputs are not modified."""
    phi, g = _d(phi), _d(g)
    w = [np.array(a, dtype=np.float64, copy=True) for a in w]
    b = [np.array(a, dtype=np.float64, copy=True) for a in b]
    D, M, N = phi.shape
    lib().orc3_wb(D, M, N, _P(p), _ptr(phi), *[_ptr(a) for a in w], *[_ptr(a) for a in b], _ptr(g))
    return tuple(w), tuple(b)


def init3(phi0):
    phi0 = _d(phi0)
    D, M, N = phi0.shape
    out = [np.empty_like(phi0) for _ in range(7)]
    lib().orc3_init(D, M, N, _ptr(phi0), *[_ptr(a) for a in out])
    return dict(phi=out[0], w=tuple(out[1:4]), b=tuple(out[4:7]))


def iterate3(p, state, g, K):
    """Advance a 3-D state dict(phi, w=(3), b=(3)) by K outer iterations, in place."""
    g = _d(g)
    state["phi"] = np.array(state["phi"], dtype=np.float64, copy=True, order="C")
    state["w"] = tuple(np.array(a, dtype=np.float64, copy=True, order="C") for a in state["w"])
    state["b"] = tuple(np.array(a, dtype=np.float64, copy=True, order="C") for a in state["b"])
    D, M, N = g.shape
    bad = lib().orc3_iterate(D, M, N, _P(p), _ptr(state["phi"]), *[_ptr(a) for a in state["w"]],
                             *[_ptr(a) for a in state["b"]], _ptr(g), K)
    if bad:
        raise FloatingPointError(f"{bad} 3-D solves failed the imaginary-part check (Q11)")
    return state


def run3(p, volume, phi0, K):
    g = edge3(volume, p["sigma"], p["rho"], p["s"])
    st = init3(phi0)
    iterate3(p, st, g, K)
    st["g"] = g
    return st
