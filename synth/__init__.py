"""Seeded synthetic-scene generator shared by the oracle tests and the CUDA path.

This module holds NONE of the PSFS method's arithmetic (no Gaussian likelihood,
no Bayes fusion, no projection-to-pixel rule).  It only builds the *inputs*
the method consumes ("given a set of images ... silhouette
likelihood maps"): calibrated pinhole cameras, a per-pixel Gaussian background
model (mu, sigma), and uint8 RGB frames rendered by exact ray casting of an
ellipsoid or a 10-cylinder body (Table 1) over a noisy
background.  Both the oracle and the GPU path consume the same bytes.
"""
from .scene import (  # noqa: F401
    CONFIGS,
    Camera,
    Grid,
    Scene,
    ring_rig,
    make_background,
    render_silhouette,
    make_frames,
    make_scene,
    skeleton_parts,
    ellipsoid_part,
)
