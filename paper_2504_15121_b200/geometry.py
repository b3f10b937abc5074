"""Rectified stereo rig, depth and triangulation (reference: geometry.py).

``StereoRig`` keeps the reference's validation (geometry.py:22-36).  The
element-wise functions on the hot path -- ``disparity_to_depth``,
``triangulate``, ``triangulate_grid``, ``depth_field`` -- run on the GPU
(csrc/sn_geometry.cu) in fp64 with the reference's operation order, so their
results equal the reference's bit for bit; they keep its signatures and
return types (numpy arrays / scalars, ``ScalarField``).
"""

from __future__ import annotations

import ctypes
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


def _run(fn_name: str, *arrays_and_args):
    from . import _native
    from ._host import current_device, stream_ptr
    dev = current_device()
    rc = getattr(_native.load(), fn_name)(_native.plan(dev.index), *arrays_and_args,
                                          stream_ptr(dev))
    _native.check(rc, fn_name)


def disparity_to_depth(d, rig: StereoRig):
    """z = fx * b / d; non-positive or non-finite disparities map to NaN
    (geometry.py:39-45).  Any shape; a 0-d input returns a numpy scalar."""
    import torch
    from . import _native
    from ._host import to_device, to_host
    arr = np.asarray(d, dtype=np.float64)
    dd = to_device(arr.reshape(-1))
    z = torch.empty_like(dd)
    rs = _native.rig_struct(rig)
    _run("sn_depth_map_f64", dd.data_ptr(), dd.numel(), ctypes.byref(rs), z.data_ptr())
    return to_host(z).reshape(arr.shape)[()]


def _shrink(full: np.ndarray, shape) -> np.ndarray:
    """The values of ``full`` (a broadcast result) over the smaller broadcast
    ``shape``: index 0 along the axes ``shape`` does not span."""
    lead = full.ndim - len(shape)
    idx = tuple(0 if i < lead else (slice(0, 1) if shape[i - lead] == 1 else slice(None))
                for i in range(full.ndim))
    return np.ascontiguousarray(full[idx]).reshape(shape)


def triangulate(u, v, d, rig: StereoRig):
    """Back-project left-image pixel (u, v) with disparity d to (x, y, z)
    (geometry.py:57-64) with numpy's broadcasting: x has the shape of
    u (+) d, y of v (+) d, z of d; 0-d results are numpy scalars."""
    import torch
    from . import _native
    from ._host import to_device, to_host
    ua, va, da = (np.asarray(a, dtype=np.float64) for a in (u, v, d))
    ub, vb, db = np.broadcast_arrays(ua, va, da)
    du, dv, dd = (to_device(np.ascontiguousarray(a).reshape(-1)) for a in (ub, vb, db))
    x, y, z = (torch.empty_like(dd) for _ in range(3))
    rs = _native.rig_struct(rig)
    _run("sn_triangulate_f64", du.data_ptr(), dv.data_ptr(), dd.data_ptr(), dd.numel(),
         ctypes.byref(rs), x.data_ptr(), y.data_ptr(), z.data_ptr())
    full = ub.shape
    xs = np.broadcast_shapes(ua.shape, da.shape)
    ys = np.broadcast_shapes(va.shape, da.shape)
    return (_shrink(to_host(x).reshape(full), xs)[()], _shrink(to_host(y).reshape(full), ys)[()],
            _shrink(to_host(z).reshape(full), da.shape)[()])


def triangulate_grid(disparity: ScalarField, rig: StereoRig) -> np.ndarray:
    """(H, W, 3) camera-space points, NaN rows where the disparity is invalid or
    non-positive (geometry.py:57-64, 85-89): one points-only pass on the GPU,
    fp64, bit-exact with the reference."""
    import torch
    from . import _native
    from ._host import to_device, to_host
    d = to_device(disparity.values)
    H, W = d.shape
    out = torch.empty((H, W, 3), dtype=torch.float64, device=d.device)
    rs = _native.rig_struct(rig)
    _run("sn_triangulate_grid_f64", d.data_ptr(), 1, H, W, ctypes.byref(rs), out.data_ptr())
    return to_host(out)


def depth_field(disparity: ScalarField, rig: StereoRig) -> ScalarField:
    """Per-pixel depth; pixels with non-positive disparity become invalid
    (geometry.py:169-172): mask = disparity.mask & isfinite(z)."""
    z = disparity_to_depth(disparity.values, rig)
    return ScalarField(z, disparity.mask & np.isfinite(z))
