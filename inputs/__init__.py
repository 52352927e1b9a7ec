"""Seeded synthetic input generators shared by the oracle and the CUDA path.

This package holds NO arithmetic of the method (no operator assembly, no TT
algebra, no solver step).  It only draws random numbers and writes down
problem data (grid sizes, cross sections, quadrature direction cosines and
weights) so that `oracle/` and `paper_2309_03347_b200/` consume identical
inputs.  See DESIGN.md "Input recipe".
"""
from .gen import *  # noqa: F401,F403
