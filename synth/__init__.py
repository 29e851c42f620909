"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

Holds NONE of the method's arithmetic (no grids, kernels, contacts or solvers):
only the seeded random draws and the five BASELINE.json configurations.  This is
the one module both ``oracle/`` (via tests) and the product harness may import.
"""
from .configs import CONFIGS, ft_test, lambda_test, layer_densities, make_config  # noqa: F401
