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
    geometry.py:169-172) in one pass from the float64 disparities, bit-exact
    fp64, computed on the GPU."""
    import torch
    from . import device
    from ._host import to_device, to_host

    d = to_device(disparity.values)
    e = torch.empty(d.shape, dtype=torch.float64, device=d.device)
    device.passable(d, rig, 1.0, edges=e)
    vals = to_host(e)
    return ScalarField(vals, ~np.isnan(vals))


def passable_set(disparity: ScalarField, rig: StereoRig, threshold: float) -> np.ndarray:
    """Boolean (H, W): edge value valid and <= threshold (decided on the
    float64 disparities)."""
    from . import device
    from ._host import to_device, to_host

    d = to_device(disparity.values)
    return to_host(device.passable(d, rig, _threshold(threshold))[0]).astype(bool)


def label_components(disparity: ScalarField, rig: StereoRig, threshold: float) -> np.ndarray:
    """int32 (H, W) labels: smallest raster index of each pixel's
    8-connected passable component, -1 elsewhere (passable set decided on the
    float64 disparities)."""
    from . import device
    from ._host import to_device, to_host

    d = to_device(disparity.values)
    return to_host(device.component_labels(d, rig, _threshold(threshold))[0])


def oriented_point_cloud(disparities, rig: StereoRig, kernel_size: int = 9,
                         threshold: float = 0.2):
    """The whole hot path on host arrays: ``disparities`` ``[B, H, W]`` (or
    ``[H, W]``), float32 or float64 -> (``[B, H, W, 6]`` float32 oriented
    points ``(x, y, z, nx, ny, nz)`` -- the dense PLY vertex record,
    cli.py:118-123 -- and ``[B, H, W]`` int32 component labels).  One C-ABI
    call (sn_pipeline_host / sn_pipeline_host_f64): chunked H2D / compute / D2H
    overlap through plan-owned pinned staging, on the device of the current
    torch context.  Other dtypes are converted to float64 (the reference's
    ScalarField type), never to float32."""
    import ctypes
    from . import _native
    from ._host import current_device
    from .kernels import KernelSpec

    d = np.asarray(disparities)
    if d.dtype != np.float32:
        d = d.astype(np.float64)
    d = np.ascontiguousarray(d)
    if d.ndim == 2:
        d = d[None]
    if d.ndim != 3:
        raise ValueError(f"disparities must have shape [B, H, W] or [H, W], got {d.shape}")
    B, H, W = d.shape
    pts = np.empty((B, H, W, 6), dtype=np.float32)
    lab = np.empty((B, H, W), dtype=np.int32)
    off = _native.offsets_array(KernelSpec.square(int(kernel_size)).offsets)
    rs = _native.rig_struct(rig)
    lib = _native.load()
    fn = lib.sn_pipeline_host if d.dtype == np.float32 else lib.sn_pipeline_host_f64
    rc = fn(_native.plan(current_device().index), d.ctypes.data, B, H, W, ctypes.byref(rs),
            off.ctypes.data, len(off), _threshold(threshold), pts.ctypes.data, None,
            lab.ctypes.data)
    _native.check(rc, "oriented_point_cloud")
    return pts, lab
