"""Fixed-pattern least-squares kernels and the convolutional estimator.

Drop-in for ``stereonorm.kernels`` (kernels.py:1-296).  Pattern validation
and the closed-form weights are host-side precomputation (once per
pattern); the per-pixel work -- masked correlation, centre correction,
border/support invalidation, closed-form normal -- runs in the fused sm_100a
pass (csrc/sn_fixed.cu) via :mod:`.device`.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._native import DegenerateSupportError
from .fields import AffineField, NormalField, ScalarField
from .geometry import StereoRig

__all__ = ["DegenerateSupportError", "KernelSpec", "PrecomputedKernels", "build_kernels",
           "convolve_affine", "estimate_normals_fixed", "estimate_affine_direct",
           "format_kernel_dump"]


@dataclass(frozen=True)
class KernelSpec:
    """Integer pixel displacements (vx, vy) relative to the observed pixel
    (kernels.py:31-55)."""

    offsets: np.ndarray

    def __post_init__(self):
        off = np.asarray(self.offsets, dtype=np.int64)
        if off.ndim != 2 or off.shape[1] != 2 or off.shape[0] == 0:
            raise ValueError("offsets must have shape (N, 2)")
        if len(np.unique(off, axis=0)) != len(off):
            raise ValueError("offsets must be distinct")
        object.__setattr__(self, "offsets", off)

    @classmethod
    def square(cls, width: int) -> "KernelSpec":
        """Centred width x width square (center included), rows top to bottom."""
        if width < 3 or width % 2 == 0:
            raise ValueError("square kernel width must be odd and >= 3")
        r = width // 2
        ys, xs = np.meshgrid(np.arange(-r, r + 1), np.arange(-r, r + 1), indexing="ij")
        return cls(np.stack([xs.ravel(), ys.ravel()], axis=1))

    def __len__(self) -> int:
        return len(self.offsets)


@dataclass(frozen=True)
class PrecomputedKernels:
    """Rows s1/s2 of (V^T V)^-1 V^T and their sums delta1/delta2
    (kernels.py:58-75)."""

    spec: KernelSpec
    alpha: float
    beta: float
    gamma: float
    det: float
    s1: np.ndarray
    s2: np.ndarray
    delta1: float
    delta2: float


def build_kernels(spec: KernelSpec, tol: float = 0.5) -> PrecomputedKernels:
    """kernels.py:78-103; raises DegenerateSupportError for collinear offsets."""
    vx = spec.offsets[:, 0].astype(np.float64)
    vy = spec.offsets[:, 1].astype(np.float64)
    alpha, beta, gamma = float(vx @ vx), float(vx @ vy), float(vy @ vy)
    det = alpha * gamma - beta * beta
    if det <= tol:
        raise DegenerateSupportError(f"offset pattern is rank deficient (det={det:g})")
    sx, sy = float(vx.sum()), float(vy.sum())
    return PrecomputedKernels(spec, alpha, beta, gamma, det,
                              (gamma * vx - beta * vy) / det, (alpha * vy - beta * vx) / det,
                              (gamma * sx - beta * sy) / det, (alpha * sy - beta * sx) / det)


def _as_kernels(kernels) -> PrecomputedKernels:
    if isinstance(kernels, PrecomputedKernels):
        return kernels
    if isinstance(kernels, KernelSpec):
        return build_kernels(kernels)
    return build_kernels(KernelSpec.square(int(kernels)))


def convolve_affine(disparity: ScalarField, kernels, threads: int | None = 1) -> AffineField:
    """Per-pixel (a1, a2) over the map, gradient convention (kernels.py:182-203);
    fp64 accumulation on the GPU."""
    from . import device
    from ._host import resolve_threads, to_device, to_host

    resolve_threads(threads)
    kern = _as_kernels(kernels)
    a1, a2, m = device.affine(to_device(disparity.values), kern)
    return AffineField(to_host(a1[0]), to_host(a2[0]), to_host(m[0]).astype(bool))


def estimate_normals_fixed(disparity: ScalarField, rig: StereoRig, kernels,
                           threads: int | None = 1) -> NormalField:
    """Dense normals from the convolutional affine fit (kernels.py:237-261),
    computed by the fused GPU pass (fp64 sums, fp32 storage)."""
    from . import device
    import torch
    from ._host import resolve_threads, to_device, to_host

    resolve_threads(threads)
    kern = _as_kernels(kernels)
    d = to_device(disparity.values)
    mask = torch.empty((1,) + tuple(d.shape), dtype=torch.uint8, device=d.device)
    out = device.oriented_points(d, rig, kern, mask=mask)
    return NormalField(to_host(out[0, ..., 3:]).astype(np.float64),
                       to_host(mask[0]).astype(bool))


def support_fit(disparity: ScalarField, u: int, v: int, offsets) -> tuple[float, float]:
    """Plain least-squares (a1, a2) at pixel (u, v) over the ``offsets`` whose
    samples are inside the frame and valid -- the single-pixel solve shared
    by estimate_affine_direct (kernels.py:206-234) and
    estimate_affine_adaptive (adaptive.py:146-174); (nan, nan) for a centre
    that is out of range or invalid, or a support with det <= 0.5.  The
    moments use the reference's column dot products, so the roundings (and
    results) are the reference's."""
    h, w = disparity.shape
    if not (0 <= v < h and 0 <= u < w) or not disparity.mask[v, u]:
        return (float("nan"), float("nan"))
    off = np.asarray(offsets)
    cols, rows = u + off[:, 0], v + off[:, 1]
    use = (cols >= 0) & (cols < w) & (rows >= 0) & (rows < h)
    use[use] &= disparity.mask[rows[use], cols[use]]
    vxy = off[use].astype(np.float64)
    dd = disparity.values[rows[use], cols[use]] - disparity.values[v, u]
    al, be, ga = (float(vxy[:, i] @ vxy[:, j]) for i, j in ((0, 0), (0, 1), (1, 1)))
    det = al * ga - be * be
    if det <= 0.5:
        return (float("nan"), float("nan"))
    b1, b2 = float(vxy[:, 0] @ dd), float(vxy[:, 1] @ dd)
    return (1.0 + (ga * b1 - be * b2) / det, (-be * b1 + al * b2) / det)


def estimate_affine_direct(disparity: ScalarField, pixel: tuple[int, int],
                           spec: KernelSpec) -> tuple[float, float]:
    """Single-pixel least-squares solve over the valid in-bounds offsets
    (kernels.py:206-234) -- a scalar diagnostic, not a per-pixel pass."""
    return support_fit(disparity, int(pixel[0]), int(pixel[1]), spec.offsets)


def format_kernel_dump(kern: PrecomputedKernels) -> str:
    """Debug listing (kernels.py:264-296): the constants, then each weight set
    as a grid when the offsets fill their bounding box, else one line per
    offset."""
    consts = {"alpha": kern.alpha, "beta": kern.beta, "gamma": kern.gamma, "det": kern.det,
              "delta1": kern.delta1, "delta2": kern.delta2}
    text = [f"offsets {len(kern.spec)}"] + [f"{k} {val:.17g}" for k, val in consts.items()]
    off = np.asarray(kern.spec.offsets)
    lo = off.min(axis=0)
    extent = off.max(axis=0) - lo + 1  # (columns, rows) of the bounding box
    boxed = len(off) == int(extent[0] * extent[1])
    for tag, weights in (("s1", kern.s1), ("s2", kern.s2)):
        text.append(f"{tag} kernel:")
        if not boxed:
            text += [f"  v=({x:+d},{y:+d})  {c:.10g}" for (x, y), c in zip(off, weights)]
            continue
        grid = np.zeros((int(extent[1]), int(extent[0])))
        grid[off[:, 1] - lo[1], off[:, 0] - lo[0]] = weights
        text += ["  vy={:+d}:  {}".format(int(lo[1]) + i, "  ".join(f"{c: .10g}" for c in row))
                 for i, row in enumerate(grid)]
    return "\n".join(text) + "\n"
