"""Seeded synthetic matching-LP inputs shared by the oracle tests, the CUDA
parity tests and bench.py.

This package holds NO arithmetic of the solver method (no scores, no
projection, no gradient, no preconditioning): it only draws the LP data
(A, b, c) following PAPER.md Appendix B ("Synthetic LP construction",
PAPER.md:673-689).  See DESIGN.md "Input recipe".
"""
from .matching import GenConfig, Instance, CONFIGS, generate, generate_shard, dest_params  # noqa: F401
