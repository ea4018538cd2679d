"""Seeded synthetic input generators shared by tests, smoke() and bench.py.

This package holds NO arithmetic of the method (Eqs. 1-5): only
weights (given data in the paper), earth models, random states and the dt
choice. Both the CUDA path and the oracle consume its output; neither imports
the other.
"""
from . import configs, fields, weights  # noqa: F401
from .configs import CONFIGS, scaled, stable_dt, weights_f32  # noqa: F401
