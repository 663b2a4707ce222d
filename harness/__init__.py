"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the paper's method (no MLP evaluation, no
stencils, no frames, no losses). It only draws points and parameters.
"""
from .gen import *  # noqa: F401,F403
