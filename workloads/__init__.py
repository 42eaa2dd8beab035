"""Seeded synthetic input generators shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the method (no projection, relaxation, inversion or
blending): it only draws scenes, cameras and boxes with the shapes and distributions of
the paper's workloads.  Both `oracle/` and
`paper_2503_00308_b200/` consume its outputs; neither imports the other.
"""
from .synth import (CONFIGS, make_config, opacity_variant, Workload, look_at_euler, random_scene,
                    nearplane_config, ties_config, stacked_config)

__all__ = ["CONFIGS", "make_config", "opacity_variant", "Workload", "look_at_euler",
           "random_scene", "nearplane_config", "ties_config", "stacked_config"]
