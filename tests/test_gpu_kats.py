"""The reference's own known-answer tests, restated on the device path.

test_geometry.py (RIG fx = fy = 1000, u0 = v0 = 0, b = 0.5):
  disparity_to_depth(100) == 5 (:30-31), invalid disparities -> NaN (:33-37),
  triangulate(u0, v0, 25) == (0, 0, 20) (:48-50), (u0+100, v0, 100) -> (0.5, 0, 5)
  (:52-54), triangulate(10, 20, 0) -> NaN (:77-79);
test_kernels.py: a tilted plane gives < 1e-3 deg (:184-192), fronto-parallel
  planes give n = (0, 0, -1) (geometry KAT :132-134 via a constant field);
test_adaptive.py (depth Laplacian, :49-75): zero on a linear depth ramp, 2.0 next
  to a 5 -> 7 depth step, invalid on the border and next to a masked sample.
The device computes points inside the fused pass and the Laplacian from
disparities, so depths are fed as d = fx b / z with values that make z exact.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _points(cuda_dev, d, rig, k=3):
    from paper_2504_15121_b200 import device
    t = torch.from_numpy(np.ascontiguousarray(d, np.float32)).to(cuda_dev)
    return device.oriented_points(t, rig, k)[0].cpu().numpy()


def test_depth_and_triangulation_kats(cuda_dev):
    from paper_2504_15121_b200 import StereoRig
    rig = StereoRig(1000.0, 1000.0, 0.0, 0.0, 0.5)
    d = np.full((4, 128), 100.0, np.float32)
    d[0, 0] = 25.0          # principal ray (u0, v0)
    d[0, 100] = 100.0       # (u0 + 100, v0)
    d[1, 10] = 0.0          # invalid disparities -> NaN point
    d[1, 11] = -3.0
    d[1, 12] = np.nan
    d[1, 13] = np.inf
    p = _points(cuda_dev, d, rig)
    assert tuple(p[0, 0, :3]) == (0.0, 0.0, 20.0)
    assert p[2, 5, 2] == 5.0
    np.testing.assert_allclose(p[0, 100, :3], (0.5, 0.0, 5.0), rtol=1e-6, atol=1e-7)
    for u in (10, 11, 12, 13):
        assert np.isnan(p[1, u, :3]).all()


def test_fronto_parallel_and_tilted_plane(cuda_dev):
    from paper_2504_15121_b200 import StereoRig, scenes
    rig = StereoRig(800.0, 800.0, 31.5, 23.5, 0.4)
    p = _points(cuda_dev, np.full((48, 64), 20.0), rig, 5)
    ok = np.isfinite(p[..., 3])
    assert ok[2:-2, 2:-2].all() and not ok[:2].any() and not ok[:, :2].any()
    np.testing.assert_allclose(p[ok][:, 3:], np.tile([0.0, 0.0, -1.0], (ok.sum(), 1)), atol=1e-6)
    n = np.array([0.25, -0.4, -1.0])
    disp, nn = scenes.plane_disparity(n / np.linalg.norm(n), -5.0, rig, 64, 48)
    p = _points(cuda_dev, disp, rig, 5)
    ok = np.isfinite(p[..., 3])
    a = p[ok][:, 3:].astype(np.float64)
    ref = n / np.linalg.norm(n)
    ang = np.degrees(np.arctan2(np.linalg.norm(np.cross(a, ref), axis=-1), np.abs(a @ ref)))
    assert ang.max() < 1e-3


def _edges(cuda_dev, z, rig):
    from paper_2504_15121_b200 import device
    d = np.where(np.isfinite(z), rig.fx * rig.baseline / z, np.nan).astype(np.float32)
    t = torch.from_numpy(d).to(cuda_dev)
    e = torch.empty(t.shape, dtype=torch.float64, device=cuda_dev)
    _, e = device.passable(t, rig, 1.0, edges=e)
    return e[0].cpu().numpy()


def test_depth_laplacian_kats(cuda_dev):
    from paper_2504_15121_b200 import StereoRig
    rig = StereoRig(35.0, 35.0, 4.5, 3.5, 1.0)  # fx b = 35: z = 5 and 7 are exact
    z = np.full((8, 10), 5.0)
    z[:, 5:] = 7.0
    e = _edges(cuda_dev, z, rig)
    np.testing.assert_allclose(e[1:-1, 4], 2.0)
    np.testing.assert_allclose(e[1:-1, 5], 2.0)
    np.testing.assert_allclose(e[1:-1, 2], 0.0)
    # border invalid
    assert np.isnan(e[0]).all() and np.isnan(e[-1]).all()
    assert np.isnan(e[:, 0]).all() and np.isnan(e[:, -1]).all()
    # a masked sample invalidates itself and its 4-neighbours
    z = np.full((7, 7), 5.0)
    z[3, 3] = np.nan
    e = _edges(cuda_dev, z, rig)
    assert np.isnan(e[3, 3]) and np.isnan(e[3, 2]) and np.isnan(e[2, 3])
    assert not np.isnan(e[1, 1])
    # zero on a linear ramp in depth -- up to the fp32 rounding of the
    # disparities d = fx b / z that carry it here (|dz| <= 2^-24 z per sample,
    # 8 samples' worth in the Laplacian: < 1e-5 for z < 10)
    v, u = np.mgrid[0:10, 0:12].astype(float)
    e = _edges(cuda_dev, 5.0 + 0.25 * u - 0.125 * v, rig)
    assert np.isfinite(e[1:-1, 1:-1]).all()
    assert np.abs(e[1:-1, 1:-1]).max() < 1e-5
