"""Passable set and connected-surface-component labels (host-facing API).

The reference has no component labeller; its adaptive
"connected surface" support is the star-fill with the ST stop
(adaptive.py:100-143), whose rays only cross pixels whose depth-Laplacian
edge value is valid and <= t (adaptive.py:80-97, 130-132).  Under ST every
star-fill support therefore lies inside one 8-connected component of that
passable set; these functions label those components on the GPU.
"""

from __future__ import annotations

import numpy as np

from .fields import ScalarField
from .geometry import StereoRig


def _threshold(t) -> float:
    t = float(t)
    if not t > 0.0:
        raise ValueError("threshold must be positive")
    return t


def edge_map(disparity: ScalarField, rig: StereoRig) -> ScalarField:
    """depth_laplacian(depth_field(disparity)) (adaptive.py:80-97,
    geometry.py:169-172), bit-exact fp64, computed on the GPU."""
    import torch
    from . import device
    from ._host import to_device, to_host

    d = to_device(disparity.values, dtype=torch.float32)
    e = torch.empty(d.shape, dtype=torch.float64, device=d.device)
    device.passable(d, rig, 1.0, edges=e)
    vals = to_host(e)
    return ScalarField(vals, np.isfinite(vals) | ~np.isnan(vals))


def passable_set(disparity: ScalarField, rig: StereoRig, threshold: float) -> np.ndarray:
    """Boolean (H, W): edge value valid and <= threshold."""
    import torch
    from . import device
    from ._host import to_device, to_host

    d = to_device(disparity.values, dtype=torch.float32)
    return to_host(device.passable(d, rig, _threshold(threshold))[0]).astype(bool)


def label_components(disparity: ScalarField, rig: StereoRig, threshold: float) -> np.ndarray:
    """int32 (H, W) labels: smallest raster index of each pixel's
    8-connected passable component, -1 elsewhere."""
    import torch
    from . import device
    from ._host import to_device, to_host

    d = to_device(disparity.values, dtype=torch.float32)
    return to_host(device.component_labels(d, rig, _threshold(threshold))[0])
