"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NO arithmetic of the method (no degrees, no Theta, no
Alg. 1 step): it only draws the hypergraph incidence H, the hyperedge weights
w and the right-hand sides Y.  The Gaussian test matrix Omega is NOT drawn
here: each side implements the same counter-based Philox4x64-10 generator
(reading A6).
"""
from .hypergraph import CONFIGS, HypergraphInput, SynthConfig, make_input, cfg5_points

__all__ = ["CONFIGS", "HypergraphInput", "SynthConfig", "make_input", "cfg5_points"]
