"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NONE of the method's arithmetic (no edge indicator, no
regularizers, no stencils, no FFT solve): it only draws images and initial
level sets with the shapes, sizes and structure of BASELINE.json's configs.
"""
from .configs import CONFIGS, make_config, paper_params, random_state  # noqa: F401
from .volumes import make_volume, paper_params3  # noqa: F401
