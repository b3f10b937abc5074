"""Adaptive star-shaped supports (ST/CD stopping) -- drop-in for the
reference's ``stereonorm.adaptive`` (adaptive.py:1-268) on the GPU.

The ray table is computed here exactly as the reference does
(``ray_offsets``, numpy ``rint`` of ``i * (cos, sin)``, adaptive.py:60-77) and
handed to the sm_100a kernel (csrc/sn_adaptive.cu) through the C ABI, which
walks the rays, builds the supports, sums the moments in the reference's
member order in fp64 and evaluates the closed-form normal.  The disparities
reach the kernel as the reference's own float64 values (no fp32 cast), so
masks and supports are bit-exact with the reference on its inputs.
``depth_laplacian`` (the ST edge measure) runs on the GPU too;
``star_trace`` and ``estimate_affine_adaptive`` are the reference's
single-pixel diagnostics, evaluated on the host ray by ray.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .fields import NormalField, ScalarField
from .geometry import StereoRig

_STOPS = ("st", "cd")

__all__ = ["StarConfig", "ray_offsets", "depth_laplacian", "estimate_normals_adaptive",
           "star_trace", "estimate_affine_adaptive"]


@dataclass(frozen=True)
class StarConfig:
    """Ray-traversal parameters (adaptive.py:32-57): ``threshold`` is the edge
    bound t for ``stop="st"`` or the covered-depth ratio k for ``stop="cd"``;
    ``shared_range`` shares one running depth range across a pixel's rays."""

    directions: int = 8
    max_steps: int = 10
    stop: str = "cd"
    threshold: float = 0.1
    shared_range: bool = False

    def __post_init__(self):
        if self.directions < 3:
            raise ValueError("need at least 3 ray directions")
        if self.max_steps < 1:
            raise ValueError("max_steps must be >= 1")
        if self.stop not in _STOPS:
            raise ValueError(f"stop must be one of {_STOPS}")
        if not self.threshold > 0.0:
            raise ValueError("threshold must be positive")


def ray_offsets(config: StarConfig) -> list[np.ndarray]:
    """Rounded integer offsets per direction, consecutive duplicates dropped
    (adaptive.py:60-77; same numpy arithmetic, so the same rounding)."""
    rays = []
    for j in range(config.directions):
        theta = 2.0 * np.pi * j / config.directions
        steps = np.arange(1, config.max_steps + 1, dtype=np.float64)
        vx = np.rint(steps * np.cos(theta)).astype(np.int64)
        vy = np.rint(steps * np.sin(theta)).astype(np.int64)
        off = np.column_stack([vx, vy])
        keep = np.ones(len(off), dtype=bool)
        keep[1:] = (off[1:] != off[:-1]).any(axis=1)
        rays.append(off[keep])
    return rays


def ray_table(config: StarConfig):
    """(lengths int32 [M], offsets int32 [sum, 2]) for the C ABI."""
    rays = ray_offsets(config)
    lens = np.array([len(r) for r in rays], dtype=np.int32)
    xy = np.ascontiguousarray(np.concatenate(rays).astype(np.int32)) if len(rays) else \
        np.zeros((0, 2), np.int32)
    return lens, xy


def depth_laplacian(depth: ScalarField) -> ScalarField:
    """5-point Laplacian magnitude of a depth field (adaptive.py:80-97), on the
    GPU in fp64 with numpy's operation order: valid only at interior pixels
    whose four neighbours are valid (mask), NaN elsewhere."""
    import torch
    from . import _native
    from ._host import current_device, stream_ptr, to_device, to_host
    z = to_device(depth.values)
    m = to_device(np.ascontiguousarray(depth.mask, dtype=np.uint8), dtype=torch.uint8)
    H, W = z.shape
    e = torch.empty_like(z)
    ok = torch.empty_like(m)
    dev = current_device()
    rc = _native.load().sn_depth_laplacian_f64(_native.plan(dev.index), z.data_ptr(),
                                               m.data_ptr(), 1, H, W, e.data_ptr(), ok.data_ptr(),
                                               stream_ptr(dev))
    _native.check(rc, "depth_laplacian")
    return ScalarField(to_host(e), to_host(ok).astype(bool))


def estimate_normals_adaptive(disparity: ScalarField, rig: StereoRig, config: StarConfig,
                              threads: int | None = 1) -> NormalField:
    """Dense normals with star-shaped adaptive supports (adaptive.py:177-268),
    computed on the GPU from the float64 disparities; masks bit-exact with
    the reference."""
    import torch
    from . import device
    from ._host import resolve_threads, to_device, to_host

    resolve_threads(threads)
    d = to_device(disparity.values)
    mask = torch.empty((1,) + tuple(d.shape), dtype=torch.uint8, device=d.device)
    out = device.adaptive_points(d, rig, config, mask=mask)
    return NormalField(to_host(out[0, ..., 3:]).astype(np.float64), to_host(mask[0]).astype(bool))


def _ray_reach(ray: np.ndarray, u: int, v: int, depth: ScalarField,
               edges: ScalarField | None, config: StarConfig, zc: float, rng):
    """Steps of one ray that the walk keeps (a prefix) and the running depth
    range after it.  ``rng`` = (rmax, rmin) entering the ray."""
    h, w = depth.shape
    xx, yy = u + ray[:, 0], v + ray[:, 1]
    inside = (xx >= 0) & (xx < w) & (yy >= 0) & (yy < h)
    xi, yi = np.where(inside, xx, 0), np.where(inside, yy, 0)
    # border and masked pixels stop the ray before any bookkeeping
    hard = inside & depth.mask[yi, xi]
    n_hard = len(ray) if hard.all() else int(np.argmin(hard))
    rmax, rmin = rng
    if config.stop == "st":
        with np.errstate(invalid="ignore"):
            ok = edges.mask[yi, xi] & ~(edges.values[yi, xi] > config.threshold)
        ok = ok[:n_hard]
        return (n_hard if ok.all() else int(np.argmin(ok))), rng
    # cd: running extremes include the step that stops the ray
    z = depth.values[yi[:n_hard], xi[:n_hard]]
    hi = np.fmax.accumulate(np.concatenate(([rmax], z)))[1:]
    lo = np.fmin.accumulate(np.concatenate(([rmin], z)))[1:]
    bad = (hi - lo) > config.threshold * zc
    n = int(np.argmax(bad)) if bad.any() else n_hard
    last = min(n, n_hard - 1)
    if last >= 0:
        rmax, rmin = max(rmax, float(hi[last])), min(rmin, float(lo[last]))
    return n, (rmax, rmin)


def star_trace(center, depth: ScalarField, edges: ScalarField | None,
               config: StarConfig) -> np.ndarray:
    """Offsets selected around one pixel, (0, 0) first and then each kept ray
    step's offset at its first occurrence (adaptive.py:100-143).  Rays stop,
    excluding the triggering pixel, at the border, at masked pixels, where the
    edge measure is invalid or exceeds t (``st``) or once the covered depth
    range exceeds t * z_c (``cd``; per ray, or shared by the pixel's rays)."""
    if config.stop == "st" and edges is None:
        raise ValueError("stop='st' requires an edge map")
    u, v = center
    h, w = depth.shape
    if not (0 <= v < h and 0 <= u < w) or not depth.mask[v, u]:
        return np.zeros((1, 2), dtype=np.int64)
    zc = float(depth.values[v, u])
    kept = [np.zeros((1, 2), dtype=np.int64)]
    rng = (zc, zc)
    for ray in ray_offsets(config):
        if config.stop == "cd" and not config.shared_range:
            rng = (zc, zc)
        n, rng = _ray_reach(ray, u, v, depth, edges, config, zc, rng)
        kept.append(ray[:n])
    steps = np.concatenate(kept).astype(np.int64)
    _, first = np.unique(steps, axis=0, return_index=True)
    return steps[np.sort(first)]


def estimate_affine_adaptive(disparity: ScalarField, depth: ScalarField,
                             edges: ScalarField | None, pixel, config: StarConfig):
    """(a1, a2) least-squares fit over one pixel's star support
    (adaptive.py:146-174): offsets with an invalid disparity sample are left
    out; (nan, nan) for an invalid centre or a rank-deficient support."""
    from .kernels import support_fit
    u, v = int(pixel[0]), int(pixel[1])
    h, w = disparity.shape
    if not (0 <= v < h and 0 <= u < w) or not disparity.mask[v, u]:
        return (float("nan"), float("nan"))
    return support_fit(disparity, u, v, star_trace((u, v), depth, edges, config))
