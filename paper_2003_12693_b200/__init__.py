"""B200-native Split Bregman solver for the Self-repelling Snake model (arXiv 2003.12693).

The product is libsrsb.so (C ABI: include/srsb.h) built from csrc/ for sm_100a;
`srsb` is its thin ctypes binding.  See DESIGN.md.
"""
from .srsb import DistSolver, Solver, Solver3, SrsbError, default_params, lib  # noqa: F401

__all__ = ["DistSolver", "Solver", "Solver3", "SrsbError", "default_params", "lib"]
