"""Adaptive star-shaped supports (ST/CD stopping) -- drop-in for the
reference's ``stereonorm.adaptive`` (adaptive.py:1-268) on the GPU.

The ray table is computed here exactly as the reference does
(``ray_offsets``, numpy ``rint`` of ``i * (cos, sin)``, adaptive.py:60-77) and
handed to the sm_100a kernel (csrc/sn_adaptive.cu) through the C ABI, which
walks the rays, builds the supports, sums the moments in the reference's
member order in fp64 and evaluates the closed-form normal.  ``star_trace`` and
``estimate_affine_adaptive`` are the reference's single-pixel diagnostics
(host, scalar), as in the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .fields import NormalField, ScalarField
from .geometry import StereoRig

_STOPS = ("st", "cd")

__all__ = ["StarConfig", "ray_offsets", "estimate_normals_adaptive", "star_trace",
           "estimate_affine_adaptive"]


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


def estimate_normals_adaptive(disparity: ScalarField, rig: StereoRig, config: StarConfig,
                              threads: int | None = 1) -> NormalField:
    """Dense normals with star-shaped adaptive supports (adaptive.py:177-268),
    computed on the GPU; masks bit-exact with the reference."""
    import torch
    from . import device
    from ._host import resolve_threads, to_device, to_host

    resolve_threads(threads)
    d = to_device(disparity.values, dtype=torch.float32)
    mask = torch.empty((1,) + tuple(d.shape), dtype=torch.uint8, device=d.device)
    out = device.adaptive_points(d, rig, config, mask=mask)
    return NormalField(to_host(out[0, ..., 3:]).astype(np.float64), to_host(mask[0]).astype(bool))


def star_trace(center, depth: ScalarField, edges: ScalarField | None,
               config: StarConfig) -> np.ndarray:
    """Offsets selected around one pixel (adaptive.py:100-143): the
    reference's single-pixel diagnostic, scalar host code."""
    if config.stop == "st" and edges is None:
        raise ValueError("stop='st' requires an edge map")
    u, v = center
    h, w = depth.shape
    selected = [(0, 0)]
    if not (0 <= v < h and 0 <= u < w) or not depth.mask[v, u]:
        return np.asarray(selected, dtype=np.int64)
    zc = depth.values[v, u]
    seen = {(0, 0)}
    rmax = rmin = zc
    for ray in ray_offsets(config):
        if config.stop == "cd" and not config.shared_range:
            rmax = rmin = zc
        for vx, vy in ray:
            uu, vv = u + vx, v + vy
            if not (0 <= uu < w and 0 <= vv < h) or not depth.mask[vv, uu]:
                break
            if config.stop == "st":
                if not edges.mask[vv, uu] or edges.values[vv, uu] > config.threshold:
                    break
            else:
                z = depth.values[vv, uu]
                rmax, rmin = max(rmax, z), min(rmin, z)
                if rmax - rmin > config.threshold * zc:
                    break
            key = (int(vx), int(vy))
            if key not in seen:
                seen.add(key)
                selected.append(key)
    return np.asarray(selected, dtype=np.int64)


def estimate_affine_adaptive(disparity: ScalarField, depth: ScalarField,
                             edges: ScalarField | None, pixel, config: StarConfig):
    """(a1, a2) over one pixel's star support (adaptive.py:146-174)."""
    u, v = pixel
    h, w = disparity.shape
    if not (0 <= v < h and 0 <= u < w) or not disparity.mask[v, u]:
        return (float("nan"), float("nan"))
    off = star_trace(pixel, depth, edges, config)
    uu, vv = u + off[:, 0], v + off[:, 1]
    ok = disparity.mask[vv, uu]
    vxy = off[ok].astype(np.float64)
    rhs = disparity.values[vv[ok], uu[ok]] - disparity.values[v, u]
    alpha, beta, gamma = float(vxy[:, 0] @ vxy[:, 0]), float(vxy[:, 0] @ vxy[:, 1]), \
        float(vxy[:, 1] @ vxy[:, 1])
    det = alpha * gamma - beta * beta
    if det <= 0.5:
        return (float("nan"), float("nan"))
    b1, b2 = float(vxy[:, 0] @ rhs), float(vxy[:, 1] @ rhs)
    return (1.0 + (gamma * b1 - beta * b2) / det, (-beta * b1 + alpha * b2) / det)
