"""Seeded synthetic input generators shared by the oracle (tests) and the product path.

This package holds NONE of the method's arithmetic (no element matrices, no
operators, no solver steps).  It only produces the inputs a user would hand
to the solver: grid sizes, per-element wavenumber arrays k_e (fine and
coarse), shift parameters (beta, sigma), the point-source right-hand side
location, and the BASELINE.json sample sweep.  Both `oracle/` and the CUDA
path consume identical bytes from here.

Readings of BASELINE.json / the paper used here are listed in DESIGN.md
(C7, C8, C9, C14-C17 of SURVEY.md section 8(c)).
"""
from .configs import (ProblemSpec, config_spec, sweep_samples, sweep_grid_n, sweep_sample_spec,
                      point_source_weights, CONFIG_NAMES)
from .media import layered_2d_velocity, inclusion_3d_velocity, element_centroids

__all__ = ["ProblemSpec", "config_spec", "sweep_samples", "sweep_grid_n", "sweep_sample_spec",
           "point_source_weights", "CONFIG_NAMES", "layered_2d_velocity",
           "inclusion_3d_velocity", "element_centroids"]
