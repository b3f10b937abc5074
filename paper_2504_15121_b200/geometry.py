"""Rectified stereo rig and triangulation (reference: geometry.py).

``StereoRig`` keeps the reference's validation (geometry.py:22-36).
``triangulate_grid`` runs on the GPU through the fused pass (the point
columns of the oriented-point record).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .fields import ScalarField


@dataclass(frozen=True)
class StereoRig:
    """Rectified camera pair: shared pin-hole intrinsics plus baseline."""

    fx: float
    fy: float
    u0: float
    v0: float
    baseline: float

    def __post_init__(self):
        if not (self.fx > 0.0 and self.fy > 0.0):
            raise ValueError("focal lengths must be positive")
        if not self.baseline > 0.0:
            raise ValueError("baseline must be positive")


def pixel_grid(height: int, width: int) -> tuple[np.ndarray, np.ndarray]:
    """(U, V) float64 coordinate grids (geometry.py:79-82)."""
    v, u = np.mgrid[0:height, 0:width]
    return u.astype(np.float64), v.astype(np.float64)


def triangulate_grid(disparity: ScalarField, rig: StereoRig) -> np.ndarray:
    """(H, W, 3) camera-space points, NaN where the disparity is invalid or
    non-positive (geometry.py:57-64, 85-89).  Computed on the GPU in fp64
    and stored as fp32 (relative error <= 1e-7)."""
    from . import device
    from ._host import to_device, to_host

    d = to_device(disparity.values)
    out = device.oriented_points(d, rig, 3)
    return to_host(out[0, ..., :3]).astype(np.float64)
