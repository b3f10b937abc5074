"""Synthetic disparity inputs (host-side, once per configuration).

Restates the reference's raycast ground truth (synth.py:22-216): analytic
spheres, axis-aligned boxes and planes in left-camera coordinates, one ray
per pixel centre with unit z so the hit parameter is the depth, nearest
positive hit wins, disparity = fx*b/z, misses are NaN.  Noise is a PCG64
normal draw over the full grid in raster order, so a (sigma, seed) pair
reproduces the reference's noisy maps bit for bit.

Also defines the SURVEY.md §8(d) workload configurations C1-C5.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .geometry import StereoRig

_EPS = 1e-9


@dataclass(frozen=True)
class Sphere:
    center: tuple
    radius: float


@dataclass(frozen=True)
class Box:
    lo: tuple
    hi: tuple


@dataclass(frozen=True)
class Plane:
    """Points P with n . P == offset (n normalised)."""

    normal: tuple
    offset: float


@dataclass
class Scene:
    rig: StereoRig
    width: int
    height: int
    primitives: list = field(default_factory=list)


def _rays(rig: StereoRig, h: int, w: int):
    v, u = np.mgrid[0:h, 0:w].astype(np.float64)
    return (u - rig.u0) / rig.fx, (v - rig.v0) / rig.fy


def _hit(prim, dx, dy):
    if isinstance(prim, Sphere):
        cx, cy, cz = prim.center
        a = dx * dx + dy * dy + 1.0
        b = -2.0 * (dx * cx + dy * cy + cz)
        c = cx * cx + cy * cy + cz * cz - prim.radius ** 2
        disc = b * b - 4.0 * a * c
        root = np.sqrt(np.maximum(disc, 0.0))
        t1 = (-b - root) / (2.0 * a)
        t2 = (-b + root) / (2.0 * a)
        t = np.where(t1 > _EPS, t1, t2)
        t = np.where((disc >= 0.0) & (t > _EPS), t, np.inf)
        n = np.stack([dx * t - cx, dy * t - cy, t - cz], axis=-1) / prim.radius
        return t, n
    if isinstance(prim, Box):
        lo = np.asarray(prim.lo, dtype=np.float64)
        hi = np.asarray(prim.hi, dtype=np.float64)
        dirs = (dx, dy, np.ones_like(dx))
        t_in = np.full(dx.shape, -np.inf)
        t_out = np.full(dx.shape, np.inf)
        axis = np.zeros(dx.shape, dtype=np.int8)
        for k in range(3):
            with np.errstate(divide="ignore", invalid="ignore"):
                ta, tb = lo[k] / dirs[k], hi[k] / dirs[k]
            near, far = np.fmin(ta, tb), np.fmax(ta, tb)
            par = dirs[k] == 0.0
            inside = (lo[k] <= 0.0) & (0.0 <= hi[k])
            near = np.where(par, -np.inf if inside else np.inf, near)
            far = np.where(par, np.inf if inside else -np.inf, far)
            axis = np.where(near > t_in, np.int8(k), axis)
            t_in = np.maximum(t_in, near)
            t_out = np.minimum(t_out, far)
        t = np.where((t_out >= t_in) & (t_in > _EPS), t_in, np.inf)
        comp = np.choose(axis, dirs)
        n = np.zeros(dx.shape + (3,))
        for k in range(3):
            n[..., k] = np.where(axis == k, -np.sign(comp), 0.0)
        return t, n
    if isinstance(prim, Plane):
        nv = np.asarray(prim.normal, dtype=np.float64)
        nv = nv / np.linalg.norm(nv)
        den = nv[0] * dx + nv[1] * dy + nv[2]
        with np.errstate(divide="ignore", invalid="ignore"):
            t = prim.offset / den
        t = np.where(np.isfinite(t) & (t > _EPS), t, np.inf)
        return t, np.broadcast_to(nv, dx.shape + (3,))
    raise TypeError(f"unknown primitive {prim!r}")


def raycast(scene: Scene):
    """Returns (disparity (H, W) float64 with NaN misses, depth, normals)."""
    h, w = scene.height, scene.width
    dx, dy = _rays(scene.rig, h, w)
    best = np.full((h, w), np.inf)
    normals = np.full((h, w, 3), np.nan)
    for prim in scene.primitives:
        t, n = _hit(prim, dx, dy)
        closer = t < best
        best = np.where(closer, t, best)
        normals = np.where(closer[..., None], n, normals)
    hit = np.isfinite(best)
    depth = np.where(hit, best, np.nan)
    pts = np.stack([dx * depth, dy * depth, depth], axis=-1)
    flip = np.sum(normals * pts, axis=-1, keepdims=True) > 0.0
    normals = np.where(flip, -normals, normals)
    normals = np.where(hit[..., None], normals, np.nan)
    disparity = scene.rig.fx * scene.rig.baseline / depth
    return disparity, depth, normals


def add_gaussian_noise(disparity: np.ndarray, sigma: float, seed: int) -> np.ndarray:
    """N(0, sigma) per pixel from PCG64(seed) in raster order over the full
    grid; invalid pixels stay NaN (synth.py:201-216)."""
    if sigma < 0.0:
        raise ValueError("sigma must be non-negative")
    d = np.asarray(disparity, dtype=np.float64)
    if sigma == 0.0:
        return d.copy()
    noise = np.random.Generator(np.random.PCG64(seed)).normal(0.0, sigma, size=d.shape)
    return np.where(np.isfinite(d), d + noise, np.nan)


def plane_disparity(normal, offset: float, rig: StereoRig, width: int, height: int):
    """Closed-form disparity of the plane n . P = offset (synth.py:174-198)."""
    n = np.asarray(normal, dtype=np.float64)
    n = n / np.linalg.norm(n)
    dx, dy = _rays(rig, height, width)
    den = n[0] * dx + n[1] * dy + n[2]
    with np.errstate(divide="ignore", invalid="ignore"):
        z = offset / den
    if not np.all(np.isfinite(z) & (z > 0.0)):
        raise ValueError("plane is not fully visible with positive depth")
    oriented = n if offset <= 0.0 else -n
    return rig.fx * rig.baseline * den / offset, np.broadcast_to(oriented, (height, width, 3))


# ---------------------------------------------------------------------------
# SURVEY.md §8(d) configurations


def street_scene(width: int = 2048, height: int = 1024, fx: float | None = None,
                 baseline: float = 0.22) -> Scene:
    """Cityscapes-like street: ground plane, two building blocks, a car-sized
    box, a far box and a back wall (C3/C4/C5)."""
    fx = float(width) if fx is None else float(fx)
    rig = StereoRig(fx=fx, fy=fx, u0=(width - 1) / 2.0, v0=(height - 1) / 2.0, baseline=baseline)
    prims = [Plane((0.0, -1.0, 0.0), -1.6), Box((-8.0, -2.0, 12.0), (-3.0, 1.6, 30.0)),
             Box((2.5, -1.0, 8.0), (4.5, 1.6, 12.0)), Box((-1.5, -0.5, 40.0), (1.5, 1.6, 44.0)),
             Plane((0.0, 0.0, -1.0), -120.0)]
    return Scene(rig, width, height, prims)


def sphere_scene(width: int = 1024, height: int = 1024, fx: float | None = None) -> Scene:
    """pkg/scenes/sphere.scn geometry (radius 1.4 at z = 3), fx scaled with width."""
    fx = float(width) if fx is None else float(fx)
    rig = StereoRig(fx=fx, fy=fx, u0=(width - 1) / 2.0, v0=(height - 1) / 2.0, baseline=0.3)
    return Scene(rig, width, height, [Sphere((0.0, 0.0, 3.0), 1.4)])


CONFIGS = {
    "C1": "640x480 tilted plane, 1 frame",
    "C2": "2888x1920 curved (sphere) surface, 1 frame",
    "C3": "2048x1024 street scene, 256 frames (sigma 0.2, seed = frame index)",
    "C4": "2048x1024 street scene, sigma 1.0 + dilated holes, 64 frames (CCL stress)",
    "C5": "7680x4320 street scene, 1 frame, 8 strips of 540 rows",
}
