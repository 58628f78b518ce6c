"""Seeded synthetic inputs (meshes, charges) used by both the oracle and the CUDA path.

Holds none of the method's arithmetic (see meshes.py header)."""
from .meshes import octasphere, icosphere, star_molecule, replicate_grid, random_rotations
from . import configs

__all__ = ["octasphere", "icosphere", "star_molecule", "replicate_grid", "random_rotations",
           "configs"]
