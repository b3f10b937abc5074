"""Device entry points on CUDA tensors (torch is plumbing: memory + streams).

Each function validates its tensors, takes the caller's current CUDA stream
and calls the C ABI (include/sn_b200.h) asynchronously -- no host
synchronisation, CUDA-graph capturable.  Shapes: disparity ``[B, H, W]`` (or
``[H, W]``), fp32 (headline path) or fp64 (the reference's own values: every
entry point has an fp64 form, so decisions are made on the unrounded
samples); outputs are allocated when not supplied.

Reference functions these replace (pkg/src/stereonorm):
  oriented_points   estimate_normals_fixed kernels.py:237-261 +
                    triangulate_grid geometry.py:85-89 (dense PLY record, cli.py:118-123)
  affine            convolve_affine kernels.py:182-203
  passable          depth_laplacian adaptive.py:80-97 + ST test adaptive.py:130-132
  component_labels  new
"""

from __future__ import annotations

import ctypes
import functools

import numpy as np
import torch

from . import _native
from ._native import check


@functools.lru_cache(maxsize=64)
def _square_offsets(width: int) -> np.ndarray:
    from .kernels import KernelSpec  # local: avoid import cycle
    off = _native.offsets_array(KernelSpec.square(width).offsets)
    off.setflags(write=False)
    return off


def _offsets_of(kernels) -> np.ndarray:
    from .kernels import PrecomputedKernels, KernelSpec  # local: avoid import cycle
    if isinstance(kernels, PrecomputedKernels):
        return _native.offsets_array(kernels.spec.offsets)
    if isinstance(kernels, KernelSpec):
        return _native.offsets_array(kernels.offsets)
    # an odd square width: the pattern is built (and validated) once per width
    return _square_offsets(int(kernels))


def _batched(disp: torch.Tensor, name: str = "disparity") -> torch.Tensor:
    if not isinstance(disp, torch.Tensor):
        raise TypeError(f"{name} must be a torch.Tensor on a CUDA device")
    if not disp.is_cuda:
        raise ValueError(f"{name} must live on a CUDA device (no CPU path exists)")
    if disp.dim() == 2:
        disp = disp.unsqueeze(0)
    if disp.dim() != 3:
        raise ValueError(f"{name} must have shape [B, H, W] or [H, W], got {tuple(disp.shape)}")
    return disp.contiguous()


def _row_pitch(d) -> int:
    """Row pitch (elements) of a CUDA tensor [B, H, W] / [H, W] whose rows are
    contiguous and evenly pitched but not packed (a column crop); 0 when the
    tensor is contiguous or not such a view."""
    if not isinstance(d, torch.Tensor) or not d.is_cuda or d.dim() not in (2, 3) \
            or d.is_contiguous() or d.dtype not in (torch.float32, torch.float64):
        return 0
    st, sh = d.stride(), d.shape
    if st[-1] != 1 or st[-2] < sh[-1]:
        return 0
    if d.dim() == 3 and sh[0] > 1 and st[0] != st[-2] * sh[-2]:
        return 0
    return int(st[-2])


def _disp_fn(d: torch.Tensor, name: str):
    """The C-ABI function for ``d``'s dtype: ``name`` (fp32) or ``name_f64``."""
    lib = _native.load()
    if d.dtype == torch.float32:
        return getattr(lib, name)
    if d.dtype == torch.float64:
        return getattr(lib, name + "_f64")
    raise ValueError(f"disparity dtype must be float32 or float64, got {d.dtype}")


def _stream(dev: torch.device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def _check_out(t: torch.Tensor | None, shape, dtype, dev, name):
    if t is None:
        return torch.empty(shape, dtype=dtype, device=dev)
    if shape[0] == 1 and tuple(t.shape) == tuple(shape[1:]):
        t = t.unsqueeze(0)  # unbatched [H, W, ...] buffer for an unbatched input
    if tuple(t.shape) != tuple(shape) or t.dtype != dtype or t.device != dev or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous {dtype} tensor of shape {tuple(shape)} on {dev}")
    return t


def oriented_points(disparity: torch.Tensor, rig, kernels=9, *, out: torch.Tensor | None = None,
                    mask: torch.Tensor | None = None, generic: bool = False,
                    row0: int = 0) -> torch.Tensor:
    """Fused fit + normal + triangulation: returns ``[B, H, W, 6]`` fp32 (always
    batched; a 2D input gives B = 1)
    ``(x, y, z, nx, ny, nz)``; NaN normals where invalid, NaN points where
    the disparity is not finite and positive.  ``mask`` (uint8 ``[B, H, W]``)
    optionally receives the normal validity.  ``row0`` is the image row of
    the first input row when the input is a strip of a taller image."""
    ld = _row_pitch(disparity)
    d = disparity.unsqueeze(0) if (ld and disparity.dim() == 2) else (
        disparity if ld else _batched(disparity))
    B, H, W = d.shape
    dev = d.device
    out = _check_out(out, (B, H, W, 6), torch.float32, dev, "out")
    if mask is not None:
        mask = _check_out(mask, (B, H, W), torch.uint8, dev, "mask")
    off = _offsets_of(kernels)
    lib = _native.load()
    if ld and not generic and not row0:
        # a row-pitched view (e.g. a crop of wider frames): no copy
        rc = _disp_fn(d, "sn_oriented_points_strided")(
            _native.plan(dev.index), d.data_ptr(), B, H, W, ld, ctypes.byref(_native.rig_struct(rig)),
            off.ctypes.data, len(off), out.data_ptr(),
            mask.data_ptr() if mask is not None else None, _stream(dev))
        check(rc, "oriented_points")
        return out
    d = d.contiguous()
    if d.dtype == torch.float32:
        fn = lib.sn_oriented_points_generic if generic else lib.sn_oriented_points
    elif d.dtype == torch.float64:
        if generic:
            raise ValueError("generic=True is an fp32 test hook")
        fn = lib.sn_oriented_points_f64
    else:
        raise ValueError(f"disparity dtype must be float32 or float64, got {d.dtype}")
    rs = _native.rig_struct(rig)
    mptr = mask.data_ptr() if mask is not None else None
    if row0:
        if generic:
            raise ValueError("row0 is not supported by the generic test hook")
        rc = _disp_fn(d, "sn_oriented_points_rows")(
            _native.plan(dev.index), d.data_ptr(), B, H, W, int(row0), ctypes.byref(rs),
            off.ctypes.data, len(off), out.data_ptr(), mptr, _stream(dev))
        check(rc, "oriented_points")
        return out
    rc = fn(_native.plan(dev.index), d.data_ptr(), B, H, W, ctypes.byref(rs), off.ctypes.data,
            len(off), out.data_ptr(), mptr, _stream(dev))
    check(rc, "oriented_points")
    return out


def bit_words(W: int) -> int:
    """uint32 words per row of a passable bit mask."""
    return (int(W) + 31) // 32


def oriented_points_bits(disparity: torch.Tensor, rig, kernels, threshold: float, *,
                         out=None, mask=None, bits=None, row0: int = 0):
    """Fused pass that also emits the ST-passable bit mask (same read of the
    disparity): returns (``[B, H, W, 6]`` fp32, ``[B, H, ceil(W/32)]`` int32
    bit words; bit ``u % 32`` of word ``u // 32`` = pixel ``u``)."""
    d = _batched(disparity)
    B, H, W = d.shape
    dev = d.device
    out = _check_out(out, (B, H, W, 6), torch.float32, dev, "out")
    if mask is not None:
        mask = _check_out(mask, (B, H, W), torch.uint8, dev, "mask")
    bits = _check_out(bits, (B, H, bit_words(W)), torch.int32, dev, "bits")
    off = _offsets_of(kernels)
    rs = _native.rig_struct(rig)
    rc = _disp_fn(d, "sn_oriented_points_bits")(
        _native.plan(dev.index), d.data_ptr(), B, H, W, int(row0), ctypes.byref(rs),
        off.ctypes.data, len(off), float(threshold), out.data_ptr(),
        mask.data_ptr() if mask is not None else None, bits.data_ptr(), _stream(dev))
    check(rc, "oriented_points_bits")
    return out, bits


def passable_bits(disparity: torch.Tensor, rig, threshold: float, *, bits=None) -> torch.Tensor:
    """ST-passable bit mask ``[B, H, ceil(W/32)]`` int32 (streaming kernel)."""
    d = _batched(disparity)
    B, H, W = d.shape
    dev = d.device
    bits = _check_out(bits, (B, H, bit_words(W)), torch.int32, dev, "bits")
    rs = _native.rig_struct(rig)
    rc = _disp_fn(d, "sn_passable_bits")(_native.plan(dev.index), d.data_ptr(), B, H, W,
                                         ctypes.byref(rs), float(threshold), bits.data_ptr(),
                                         _stream(dev))
    check(rc, "passable_bits")
    return bits


def labels_from_bits(bits: torch.Tensor, width: int, *, out=None, row_base: int = 0,
                     workspace: torch.Tensor | None = None) -> torch.Tensor:
    """Component labels from a passable bit mask ``[B, H, ceil(W/32)]``."""
    bits = _batched(bits, "bits")
    if bits.dtype != torch.int32 or bits.shape[-1] != bit_words(width):
        raise ValueError("bits must be int32 [B, H, ceil(width/32)]")
    B, H, _ = bits.shape
    W = int(width)
    dev = bits.device
    out = _check_out(out, (B, H, W), torch.int32, dev, "out")
    ws = _workspace(workspace, B, H, W, dev)
    rc = _native.load().sn_ccl_from_bits_ws(_native.plan(dev.index), bits.data_ptr(), B, H, W,
                                            int(row_base), out.data_ptr(), ws.data_ptr(),
                                            ws.numel() * ws.element_size(), _stream(dev))
    check(rc, "labels_from_bits")
    return out


def pipeline(disparity: torch.Tensor, rig, kernels, threshold: float, *, out=None, labels=None,
             mask=None, workspace: torch.Tensor | None = None):
    """The whole hot path in one call: fused fit + normal + point + passable
    bits, then component labels.  Returns (``[B, H, W, 6]`` fp32, ``[B, H, W]``
    int32 labels)."""
    d = _batched(disparity)
    B, H, W = d.shape
    dev = d.device
    out = _check_out(out, (B, H, W, 6), torch.float32, dev, "out")
    labels = _check_out(labels, (B, H, W), torch.int32, dev, "labels")
    if mask is not None:
        mask = _check_out(mask, (B, H, W), torch.uint8, dev, "mask")
    ws = _workspace(workspace, B, H, W, dev)
    off = _offsets_of(kernels)
    rs = _native.rig_struct(rig)
    rc = _disp_fn(d, "sn_pipeline_ws")(
        _native.plan(dev.index), d.data_ptr(), B, H, W, ctypes.byref(rs), off.ctypes.data,
        len(off), float(threshold), out.data_ptr(), mask.data_ptr() if mask is not None else None,
        labels.data_ptr(), ws.data_ptr(), ws.numel() * ws.element_size(), _stream(dev))
    check(rc, "pipeline")
    return out, labels


def adaptive_points(disparity: torch.Tensor, rig, config, *, out=None, mask=None,
                    workspace: torch.Tensor | None = None) -> torch.Tensor:
    """Adaptive star-fill pass (adaptive.py:177-268): ``[B, H, W, 6]`` fp32
    records with normals over edge-aware star supports (``config`` a
    ``StarConfig``); ``mask`` (uint8) optionally receives the validity."""
    from .adaptive import ray_table
    d = _batched(disparity)
    B, H, W = d.shape
    dev = d.device
    out = _check_out(out, (B, H, W, 6), torch.float32, dev, "out")
    if mask is not None:
        mask = _check_out(mask, (B, H, W), torch.uint8, dev, "mask")
    n = ctypes.c_size_t(0)
    lib = _native.load()
    check(lib.sn_adaptive_workspace_bytes(B, H, W, ctypes.byref(n)), "sn_adaptive_workspace_bytes")
    if workspace is None:
        workspace = torch.empty(max(1, n.value), dtype=torch.uint8, device=dev)
    elif workspace.numel() * workspace.element_size() < n.value or workspace.device != dev:
        raise ValueError(f"workspace must hold >= {n.value} bytes on {dev}")
    lens, xy = ray_table(config)
    rs = _native.rig_struct(rig)
    rc = _disp_fn(d, "sn_adaptive_points")(_native.plan(dev.index), d.data_ptr(), B, H, W, ctypes.byref(rs),
                                len(lens), lens.ctypes.data, xy.ctypes.data,
                                0 if config.stop == "st" else 1, int(bool(config.shared_range)),
                                float(config.threshold), out.data_ptr(),
                                mask.data_ptr() if mask is not None else None,
                                workspace.data_ptr(), workspace.numel() * workspace.element_size(),
                                _stream(dev))
    check(rc, "adaptive_points")
    return out


def angular_error(est: torch.Tensor, gt: torch.Tensor, gt_mask: torch.Tensor, *, mask=None,
                  want_map: bool = True):
    """Device accuracy evaluation (evaluation.py:34-73): ``est`` is either the
    dense record ``[B, H, W, 6]`` (fp32) or normals ``[B, H, W, 3]`` (fp32 or
    fp64, NaN = invalid); ``gt`` fp64 ``[B, H, W, 3]`` with ``gt_mask`` (bool /
    uint8).  Returns (angle map fp64 ``[B, H, W]`` NaN-invalid or None,
    stats fp64 ``[B, 6]`` = avg, min, max, lower median, population std, count)."""
    if est.dim() == 3:
        est, gt, gt_mask = est.unsqueeze(0), gt.unsqueeze(0), gt_mask.unsqueeze(0)
        mask = mask.unsqueeze(0) if mask is not None else None
    if est.dim() != 4 or est.shape[-1] not in (3, 6):
        raise ValueError("est must be [B, H, W, 6] records or [B, H, W, 3] normals")
    est = est.contiguous()
    B, H, W, stride = est.shape
    dev = est.device
    if est.dtype == torch.float64 and stride != 3:
        raise ValueError("fp64 est must be [B, H, W, 3] normals")
    gt = _check_out(gt.contiguous(), (B, H, W, 3), torch.float64, dev, "gt")
    gm = gt_mask.to(torch.uint8).contiguous()
    em = mask.to(torch.uint8).contiguous() if mask is not None else None
    n = ctypes.c_size_t(0)
    lib = _native.load()
    check(lib.sn_eval_workspace_bytes(B, H, W, ctypes.byref(n)), "sn_eval_workspace_bytes")
    ws = torch.empty(max(1, n.value), dtype=torch.uint8, device=dev)
    err = torch.empty((B, H, W), dtype=torch.float64, device=dev) if want_map else None
    stats = torch.empty((B, 6), dtype=torch.float64, device=dev)
    fn = lib.sn_angular_error_f64 if est.dtype == torch.float64 else lib.sn_angular_error
    if est.dtype not in (torch.float32, torch.float64):
        raise ValueError("est must be float32 or float64")
    rc = fn(_native.plan(dev.index), est.data_ptr(), stride, gt.data_ptr(), gm.data_ptr(),
            em.data_ptr() if em is not None else None, B, H, W,
            err.data_ptr() if err is not None else None, stats.data_ptr(), ws.data_ptr(),
            n.value, _stream(dev))
    check(rc, "angular_error")
    return err, stats


def error_stats(values: torch.Tensor) -> torch.Tensor:
    """summarize (evaluation.py:58-73) of fp64 maps ``[B, H, W]`` (non-finite =
    invalid): ``[B, 6]`` = avg, min, max, lower median, population std, count."""
    v = _batched(values, "values")
    if v.dtype != torch.float64:
        raise ValueError("values must be float64")
    B, H, W = v.shape
    dev = v.device
    n = ctypes.c_size_t(0)
    lib = _native.load()
    check(lib.sn_eval_workspace_bytes(B, H, W, ctypes.byref(n)), "sn_eval_workspace_bytes")
    ws = torch.empty(max(1, n.value), dtype=torch.uint8, device=dev)
    stats = torch.empty((B, 6), dtype=torch.float64, device=dev)
    rc = lib.sn_error_stats(_native.plan(dev.index), v.data_ptr(), B, H, W, stats.data_ptr(),
                            ws.data_ptr(), n.value, _stream(dev))
    check(rc, "error_stats")
    return stats


def compact_cloud(records: torch.Tensor, mask: torch.Tensor):
    """Stream-compact the dense ``[B, H, W, 6]`` records of pixels with a valid
    normal (``mask`` uint8 ``[B, H, W]`` from ``oriented_points(..., mask=)``)
    into ``[N, 6]`` float32 vertices in raster order -- the binary-PLY body
    (cli.py:118-123, formats.py:170-185).  Returns (vertices, offsets): frame f
    owns ``vertices[offsets[f]:offsets[f+1]]`` (offsets int64 ``[B+1]``, host)."""
    if records.dim() == 3:
        records = records.unsqueeze(0)
    if records.dim() != 4 or records.shape[-1] != 6 or records.dtype != torch.float32:
        raise ValueError("records must be float32 [B, H, W, 6]")
    records = records.contiguous()
    B, H, W, _ = records.shape
    dev = records.device
    mask = _check_out(mask, (B, H, W), torch.uint8, dev, "mask")
    n = ctypes.c_size_t(0)
    check(_native.load().sn_cloud_workspace_bytes(B, H, W, ctypes.byref(n)), "sn_cloud_workspace_bytes")
    ws = torch.empty(max(1, n.value), dtype=torch.uint8, device=dev)
    offsets = torch.empty(B + 1, dtype=torch.int64, device=dev)
    lib = _native.load()

    plan = _native.plan(dev.index)
    # count + scan, read the total back to size the output, then scatter
    check(lib.sn_cloud_count(plan, mask.data_ptr(), B, H, W, offsets.data_ptr(), ws.data_ptr(),
                             n.value, _stream(dev)), "compact_cloud")
    total = int(offsets[B].item())
    cloud = torch.empty((total, 6), dtype=torch.float32, device=dev)
    if total:
        check(lib.sn_cloud_scatter(plan, records.data_ptr(), mask.data_ptr(), B, H, W,
                                   cloud.data_ptr(), total, ws.data_ptr(), n.value, _stream(dev)),
              "compact_cloud")
    return cloud, offsets.cpu()


def _raw16(raw: torch.Tensor) -> torch.Tensor:
    if raw.dtype not in (torch.uint16, torch.int16):
        raise ValueError(f"PNG16 samples must be uint16 (or int16 bits), got {raw.dtype}")
    if raw.dim() == 2:
        raw = raw.unsqueeze(0)
    if raw.dim() != 3:
        raise ValueError("PNG16 samples must be [H, W] or [B, H, W]")
    if not raw.is_cuda:
        raise ValueError("PNG16 samples must be on a CUDA device")
    return raw.contiguous()


def _invalid16(invalid_value) -> int:
    return -1 if invalid_value is None else int(invalid_value)


def dequant_png16(raw: torch.Tensor, scale: float = 256.0, invalid_value: int | None = 0, *,
                  dtype=torch.float64, out=None) -> torch.Tensor:
    """read_disparity_png16's sample step (formats.py:133-150) on the device:
    ``d = (raw - 1) / scale`` in fp64, ``raw == invalid_value`` -> NaN.
    float64 output is the reference's value bit for bit, float32 that value
    rounded once.  Returns ``[B, H, W]``."""
    r = _raw16(raw)
    B, H, W = r.shape
    dev = r.device
    if dtype not in (torch.float32, torch.float64):
        raise ValueError("dtype must be float32 or float64")
    out = _check_out(out, (B, H, W), dtype, dev, "out")
    p32 = out.data_ptr() if dtype == torch.float32 else None
    p64 = out.data_ptr() if dtype == torch.float64 else None
    rc = _native.load().sn_dequant_png16(_native.plan(dev.index), r.data_ptr(), B, H, W,
                                         float(scale), _invalid16(invalid_value), p32, p64,
                                         _stream(dev))
    check(rc, "dequant_png16")
    return out


def decode_pfm(payload: torch.Tensor, height: int, width: int, channels: int = 1,
               big_endian: bool = False, *, out=None) -> torch.Tensor:
    """The PFM payload step (formats.py:84-102) on the device: ``payload`` is
    ``[B, H*W*C*4]`` (or flat) uint8 bytes of B images, bottom row first;
    returns native float32 ``[B, H, W]`` (``[B, H, W, 3]`` for C = 3), top row
    first."""
    if payload.dtype != torch.uint8 or not payload.is_cuda:
        raise ValueError("payload must be a CUDA uint8 tensor")
    per = int(height) * int(width) * int(channels) * 4
    flat = payload.contiguous().reshape(-1)
    if per == 0 or flat.numel() % per:
        raise ValueError(f"payload of {flat.numel()} bytes is not a whole number of "
                         f"{height}x{width}x{channels} PFM images")
    B = flat.numel() // per
    dev = flat.device
    shape = (B, height, width) + ((3,) if channels == 3 else ())
    out = _check_out(out, shape, torch.float32, dev, "out")
    rc = _native.load().sn_decode_pfm(_native.plan(dev.index), flat.data_ptr(), B, int(height),
                                      int(width), int(channels), 1 if big_endian else 0,
                                      out.data_ptr(), _stream(dev))
    check(rc, "decode_pfm")
    return out


def oriented_points_png16(raw: torch.Tensor, rig, kernels=9, *, scale: float = 256.0,
                          invalid_value: int | None = 0, out=None, mask=None) -> torch.Tensor:
    """``oriented_points`` reading 16-bit PNG samples directly (2 B/px): the
    fused pass dequantises on load exactly as read_disparity_png16 does.
    Needs a centred square kernel and 2^-100 <= |scale| <= 2^100."""
    r = _raw16(raw)
    B, H, W = r.shape
    dev = r.device
    out = _check_out(out, (B, H, W, 6), torch.float32, dev, "out")
    if mask is not None:
        mask = _check_out(mask, (B, H, W), torch.uint8, dev, "mask")
    off = _offsets_of(kernels)
    rs = _native.rig_struct(rig)
    rc = _native.load().sn_oriented_points_png16(
        _native.plan(dev.index), r.data_ptr(), B, H, W, float(scale), _invalid16(invalid_value),
        ctypes.byref(rs), off.ctypes.data, len(off), out.data_ptr(),
        mask.data_ptr() if mask is not None else None, _stream(dev))
    check(rc, "oriented_points_png16")
    return out


def affine(disparity: torch.Tensor, kernels, *, a1=None, a2=None, mask=None):
    """convolve_affine on the device: (a1, a2, mask) fp64/fp64/uint8 ``[B, H, W]``."""
    d = _batched(disparity)
    B, H, W = d.shape
    dev = d.device
    a1 = _check_out(a1, (B, H, W), torch.float64, dev, "a1")
    a2 = _check_out(a2, (B, H, W), torch.float64, dev, "a2")
    mask = _check_out(mask, (B, H, W), torch.uint8, dev, "mask")
    off = _offsets_of(kernels)
    lib = _native.load()
    if d.dtype == torch.float32:
        fn = lib.sn_affine
    elif d.dtype == torch.float64:
        fn = lib.sn_affine_f64
    else:
        raise ValueError(f"disparity dtype must be float32 or float64, got {d.dtype}")
    rc = fn(_native.plan(dev.index), d.data_ptr(), B, H, W, off.ctypes.data, len(off),
            a1.data_ptr(), a2.data_ptr(), mask.data_ptr(), _stream(dev))
    check(rc, "affine")
    return a1, a2, mask


def passable(disparity: torch.Tensor, rig, threshold: float, *, out=None, edges=None):
    """ST-passable set (uint8) and optionally the depth-Laplacian values."""
    d = _batched(disparity)
    B, H, W = d.shape
    dev = d.device
    out = _check_out(out, (B, H, W), torch.uint8, dev, "out")
    want_edges = edges is not None
    if want_edges:
        edges = _check_out(edges, (B, H, W), torch.float64, dev, "edges")
    rs = _native.rig_struct(rig)
    rc = _disp_fn(d, "sn_passable")(_native.plan(dev.index), d.data_ptr(), B, H, W,
                                    ctypes.byref(rs), float(threshold), out.data_ptr(),
                                    edges.data_ptr() if want_edges else None, _stream(dev))
    check(rc, "passable")
    return (out, edges) if want_edges else out


def ccl_workspace(B: int, H: int, W: int, dev: torch.device) -> torch.Tensor:
    """Device scratch for the labeller (bit mask + tile seams), from torch's
    caching allocator so concurrent streams never share one."""
    return torch.empty(_native.ccl_workspace_bytes(B, H, W), dtype=torch.uint8, device=dev)


def _workspace(ws, B, H, W, dev):
    need = _native.ccl_workspace_bytes(B, H, W)
    if ws is None:
        return torch.empty(need, dtype=torch.uint8, device=dev)
    if ws.device != dev or not ws.is_contiguous() or ws.numel() * ws.element_size() < need:
        raise ValueError(f"workspace must be a contiguous buffer of >= {need} bytes on {dev}")
    return ws


def component_labels(disparity: torch.Tensor, rig, threshold: float, *, out=None,
                     row_base: int = 0, workspace: torch.Tensor | None = None) -> torch.Tensor:
    """8-connected labels of the ST-passable set: int32 ``[B, H, W]`` holding
    the smallest raster index ``v*W + u`` (+ ``row_base*W``) of each pixel's
    component, -1 where not passable."""
    d = _batched(disparity)
    B, H, W = d.shape
    dev = d.device
    out = _check_out(out, (B, H, W), torch.int32, dev, "out")
    ws = _workspace(workspace, B, H, W, dev)
    rs = _native.rig_struct(rig)
    rc = _disp_fn(d, "sn_ccl_labels_ws")(_native.plan(dev.index), d.data_ptr(), B, H, W,
                                         ctypes.byref(rs), float(threshold), int(row_base),
                                         out.data_ptr(), ws.data_ptr(),
                                         ws.numel() * ws.element_size(), _stream(dev))
    check(rc, "component_labels")
    return out


def labels_from_passable(p: torch.Tensor, *, out=None, row_base: int = 0,
                         workspace: torch.Tensor | None = None) -> torch.Tensor:
    """Label an existing uint8/bool passable grid ``[B, H, W]``."""
    p = _batched(p, "passable")
    if p.dtype == torch.bool:
        p = p.to(torch.uint8)
    if p.dtype != torch.uint8:
        raise ValueError("passable must be uint8 or bool")
    B, H, W = p.shape
    dev = p.device
    out = _check_out(out, (B, H, W), torch.int32, dev, "out")
    ws = _workspace(workspace, B, H, W, dev)
    rc = _native.load().sn_ccl_from_passable_ws(_native.plan(dev.index), p.data_ptr(), B, H, W,
                                                int(row_base), out.data_ptr(), ws.data_ptr(),
                                                ws.numel() * ws.element_size(), _stream(dev))
    check(rc, "labels_from_passable")
    return out


def relabel(labels: torch.Tensor, keys: torch.Tensor, vals: torch.Tensor, n_map: torch.Tensor,
            index_base: int, scratch: torch.Tensor | None = None) -> torch.Tensor:
    """In-place (label -> root) remap of one strip's labels (device)."""
    if not labels.is_cuda or labels.dtype != torch.int32 or not labels.is_contiguous():
        raise ValueError("labels must be a contiguous int32 CUDA tensor")
    dev = labels.device
    n = labels.numel()
    if scratch is None:
        scratch = torch.empty(n, dtype=torch.int32, device=dev)
    rc = _native.load().sn_relabel(_native.plan(dev.index), labels.data_ptr(), n, int(index_base),
                                   keys.data_ptr(), vals.data_ptr(), n_map.data_ptr(),
                                   int(keys.numel()), scratch.data_ptr(), _stream(dev))
    check(rc, "relabel")
    return labels


def seam_merge(seams: np.ndarray):
    """Deterministic union-find over gathered seam rows (host, tiny).
    ``seams``: int32 ``[n_strips, 2, W]``.  Returns (keys, vals) int32."""
    s = np.ascontiguousarray(np.asarray(seams, dtype=np.int32))
    if s.ndim != 3 or s.shape[1] != 2:
        raise ValueError("seams must have shape [n_strips, 2, W]")
    n_strips, _, W = s.shape
    cap = max(1, 2 * n_strips * W)
    keys = np.empty(cap, dtype=np.int32)
    vals = np.empty(cap, dtype=np.int32)
    n = ctypes.c_int32(0)
    rc = _native.load().sn_seam_merge_host(s.ctypes.data, n_strips, W, keys.ctypes.data,
                                           vals.ctypes.data, ctypes.byref(n))
    check(rc, "seam_merge")
    return keys[:n.value].copy(), vals[:n.value].copy()


def seam_table(seams: torch.Tensor, table_n: int, *, table=None) -> torch.Tensor:
    """Device seam merge (sn_seam_merge): ``seams`` int32 ``[n_strips, 2, W]``
    on the device (the gathered first/last owned label rows); returns the
    int32 table of ``table_n`` entries mapping every seam label to its root
    (-1 elsewhere) -- identical on every rank, no host round trip."""
    if not seams.is_cuda or seams.dtype != torch.int32 or seams.dim() != 3 or seams.shape[1] != 2:
        raise ValueError("seams must be an int32 CUDA tensor [n_strips, 2, W]")
    seams = seams.contiguous()
    dev = seams.device
    table = _check_out(table, (int(table_n),), torch.int32, dev, "table")
    n_strips, _, W = seams.shape
    rc = _native.load().sn_seam_merge(_native.plan(dev.index), seams.data_ptr(), n_strips, W,
                                      table.data_ptr(), int(table_n), _stream(dev))
    check(rc, "seam_table")
    return table


def relabel_table(labels: torch.Tensor, table: torch.Tensor) -> torch.Tensor:
    """In place: every label v >= 0 with table[v] >= 0 becomes table[v]."""
    if not labels.is_cuda or labels.dtype != torch.int32 or not labels.is_contiguous():
        raise ValueError("labels must be a contiguous int32 CUDA tensor")
    if table.dtype != torch.int32 or table.device != labels.device:
        raise ValueError("table must be an int32 tensor on the labels' device")
    dev = labels.device
    rc = _native.load().sn_relabel_table(_native.plan(dev.index), labels.data_ptr(), labels.numel(),
                                         table.data_ptr(), table.numel(), _stream(dev))
    check(rc, "relabel_table")
    return labels
