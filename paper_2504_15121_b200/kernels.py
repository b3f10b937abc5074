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


def estimate_affine_direct(disparity: ScalarField, pixel: tuple[int, int],
                           spec: KernelSpec) -> tuple[float, float]:
    """Single-pixel least-squares solve over the valid in-bounds offsets
    (kernels.py:206-234) -- a scalar diagnostic, not a per-pixel pass."""
    u, v = pixel
    h, w = disparity.shape
    if not (0 <= v < h and 0 <= u < w) or not disparity.mask[v, u]:
        return (float("nan"), float("nan"))
    uu = u + spec.offsets[:, 0]
    vv = v + spec.offsets[:, 1]
    inside = (uu >= 0) & (uu < w) & (vv >= 0) & (vv < h)
    keep = inside.copy()
    keep[inside] = disparity.mask[vv[inside], uu[inside]]
    off = spec.offsets[keep].astype(np.float64)
    rhs = disparity.values[vv[keep], uu[keep]] - disparity.values[v, u]
    a, b, g = off[:, 0] @ off[:, 0], off[:, 0] @ off[:, 1], off[:, 1] @ off[:, 1]
    det = a * g - b * b
    if det <= 0.5:
        return (float("nan"), float("nan"))
    b1, b2 = off[:, 0] @ rhs, off[:, 1] @ rhs
    return (1.0 + (g * b1 - b * b2) / det, (a * b2 - b * b1) / det)


def format_kernel_dump(kern: PrecomputedKernels) -> str:
    """Debug listing: constants, then weights as grids for box-filling
    patterns or one line per offset otherwise (kernels.py:264-296)."""
    out = [f"offsets {len(kern.spec)}"]
    for name in ("alpha", "beta", "gamma", "det", "delta1", "delta2"):
        out.append(f"{name} {getattr(kern, name):.17g}")
    off = kern.spec.offsets
    x0, y0 = off[:, 0].min(), off[:, 1].min()
    nx, ny = off[:, 0].max() - x0 + 1, off[:, 1].max() - y0 + 1
    dense = len(off) == nx * ny
    for name, wts in (("s1", kern.s1), ("s2", kern.s2)):
        out.append(f"{name} kernel:")
        if dense:
            grid = np.zeros((ny, nx))
            grid[off[:, 1] - y0, off[:, 0] - x0] = wts
            for i in range(ny):
                cells = "  ".join(f"{c: .10g}" for c in grid[i])
                out.append(f"  vy={y0 + i:+d}:  {cells}")
        else:
            out.extend(f"  v=({x:+d},{y:+d})  {c:.10g}" for (x, y), c in zip(off, wts))
    return "\n".join(out) + "\n"
