"""Seeded synthetic inputs shared by the CUDA path and the CPU oracle.

This package holds NO arithmetic of the method (no DFT, no distances, no
filtering, no eigen-solving, no FD assembly). It only draws Gaussian random
fields and evaluates the PDE coefficient functions at grid nodes and face
midpoints, following the recipe stated in DESIGN.md §3.
Both sides consume the arrays it produces; neither side imports the other.
"""
from .configs import CONFIGS, Config, get_config
from .grf import OperatorFields, make_fields, make_batch, make_perturbed, grf_std, constant_fields, draw_xi

__all__ = ["CONFIGS", "Config", "get_config", "OperatorFields", "make_fields", "make_perturbed",
           "make_batch", "grf_std", "constant_fields", "draw_xi"]
