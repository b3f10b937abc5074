"""stereonorm-b200: B200-native per-pixel surface normals + oriented points.

Drop-in for the hot path of the reference package ``stereonorm`` 0.1.0
(arXiv 2504.15121): disparity -> fixed-kernel affine least squares
("convolution-style robust denoising") -> closed-form normal + triangulated
point -> ST-passable connected-surface-component labels -> dense oriented
point cloud.  The reference's public names on that path are re-exported with
identical signatures; the per-pixel work runs in hand-written sm_100a CUDA
(``csrc/``) through the C ABI in ``include/sn_b200.h``.  There is no CPU
fallback: without the built library every hot-path call raises.

Device-resident batches use :mod:`paper_2504_15121_b200.device` (torch CUDA
tensors, [B, H, W] in, [B, H, W, 6] fp32 out); multi-GPU sharding lives in
:mod:`paper_2504_15121_b200.parallel`.
"""

from ._native import DegenerateSupportError, NativeLibraryError
from .components import edge_map, label_components, oriented_point_cloud, passable_set
from .adaptive import (StarConfig, depth_laplacian, estimate_affine_adaptive,
                       estimate_normals_adaptive, ray_offsets, star_trace)
from .estimators import (AdaptiveNormalEstimator, AffineNormalEstimator, BaseNormalEstimator,
                         as_rig, as_scalar_field)
from .evaluation import ErrorStats, angular_error_map, error_stats, summarize
from .fields import AffineField, NormalField, ScalarField
from .formats import (FormatError, read_disparity_png16, read_pfm, read_pfm_normals,
                      write_disparity_png16, write_pfm, write_pfm_normals)
from .geometry import (StereoRig, depth_field, disparity_to_depth, pixel_grid, triangulate,
                       triangulate_grid)
from .kernels import (KernelSpec, PrecomputedKernels, build_kernels, convolve_affine,
                      estimate_affine_direct, estimate_normals_fixed, format_kernel_dump)

__version__ = "0.1.0"

__all__ = [
    "AdaptiveNormalEstimator", "ErrorStats", "angular_error_map", "error_stats", "summarize", "AffineField", "AffineNormalEstimator", "StarConfig",
    "estimate_affine_adaptive", "estimate_normals_adaptive", "ray_offsets", "star_trace",
    "depth_laplacian", "depth_field", "disparity_to_depth", "triangulate",
    "BaseNormalEstimator", "DegenerateSupportError",
    "FormatError", "read_disparity_png16", "read_pfm", "read_pfm_normals",
    "write_disparity_png16", "write_pfm", "write_pfm_normals",
    "KernelSpec", "NativeLibraryError", "NormalField", "PrecomputedKernels", "ScalarField",
    "StereoRig", "as_rig", "as_scalar_field", "build_kernels", "convolve_affine", "edge_map",
    "estimate_affine_direct", "estimate_normals_fixed", "format_kernel_dump",
    "label_components", "oriented_point_cloud", "passable_set", "pixel_grid", "triangulate_grid",
]
