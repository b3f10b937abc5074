"""ctypes binding of the in-tree C-ABI library ``libsn_b200.so``.

The library is built by ``__graft_entry__.build()`` (or ``make -C
paper_2504_15121_b200/csrc``) for sm_100a.  There is no CPU fallback: if the
library is missing every hot-path call raises :class:`NativeLibraryError`.
Return codes map onto the reference's exception types:
SN_EINVAL -> ValueError, SN_EDEGENERATE -> DegenerateSupportError,
SN_ECUDA -> RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libsn_b200.so"

SN_OK, SN_EINVAL, SN_EDEGENERATE, SN_ECUDA = 0, 1, 2, 3


class NativeLibraryError(RuntimeError):
    """The CUDA library is not built / not loadable (no CPU fallback exists)."""


class DegenerateSupportError(ValueError):
    """Offset pattern spans less than two independent directions
    (reference: kernels.py:27-28)."""


class SnRig(ctypes.Structure):
    _fields_ = [("fx", ctypes.c_double), ("fy", ctypes.c_double), ("u0", ctypes.c_double),
                ("v0", ctypes.c_double), ("baseline", ctypes.c_double)]


class SnMoments(ctypes.Structure):
    _fields_ = [("alpha", ctypes.c_int64), ("beta", ctypes.c_int64), ("gamma", ctypes.c_int64),
                ("det", ctypes.c_int64), ("sx", ctypes.c_int64), ("sy", ctypes.c_int64),
                ("hx", ctypes.c_int32), ("hy", ctypes.c_int32), ("square_r", ctypes.c_int32)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_D = ctypes.c_double
_RIGP = ctypes.POINTER(SnRig)

# name -> argtypes (every function returns int unless listed in _RESTYPES)
SIGNATURES = {
    "sn_abi_version": [],
    "sn_last_error": [],
    "sn_plan_create": [ctypes.c_int, ctypes.POINTER(_P)],
    "sn_plan_destroy": [_P],
    "sn_kernel_moments": [_P, _I32, ctypes.POINTER(SnMoments)],
    "sn_oriented_points": [_P, _P, _I64, _I64, _I64, _RIGP, _P, _I32, _P, _P, _P],
    "sn_oriented_points_f64": [_P, _P, _I64, _I64, _I64, _RIGP, _P, _I32, _P, _P, _P],
    "sn_oriented_points_generic": [_P, _P, _I64, _I64, _I64, _RIGP, _P, _I32, _P, _P, _P],
    "sn_oriented_points_strided": [_P, _P, _I64, _I64, _I64, _I64, _RIGP, _P, _I32, _P, _P, _P],
    "sn_oriented_points_strided_f64": [_P, _P, _I64, _I64, _I64, _I64, _RIGP, _P, _I32, _P, _P,
                                       _P],
    "sn_oriented_points_rows": [_P, _P, _I64, _I64, _I64, _I64, _RIGP, _P, _I32, _P, _P, _P],
    "sn_oriented_points_bits": [_P, _P, _I64, _I64, _I64, _I64, _RIGP, _P, _I32, _D, _P, _P, _P,
                                _P],
    "sn_passable_bits": [_P, _P, _I64, _I64, _I64, _RIGP, _D, _P, _P],
    "sn_passable_bits_f64": [_P, _P, _I64, _I64, _I64, _RIGP, _D, _P, _P],
    "sn_oriented_points_bits_f64": [_P, _P, _I64, _I64, _I64, _I64, _RIGP, _P, _I32, _D, _P, _P,
                                    _P, _P],
    "sn_oriented_points_rows_f64": [_P, _P, _I64, _I64, _I64, _I64, _RIGP, _P, _I32, _P, _P, _P],
    "sn_adaptive_points_f64": [_P, _P, _I64, _I64, _I64, _RIGP, _I32, _P, _P, _I32, _I32, _D, _P,
                               _P, _P, ctypes.c_size_t, _P],
    "sn_pipeline_f64": [_P, _P, _I64, _I64, _I64, _RIGP, _P, _I32, _D, _P, _P, _P, _P],
    "sn_pipeline_ws_f64": [_P, _P, _I64, _I64, _I64, _RIGP, _P, _I32, _D, _P, _P, _P, _P,
                           ctypes.c_size_t, _P],
    "sn_passable_f64": [_P, _P, _I64, _I64, _I64, _RIGP, _D, _P, _P, _P],
    "sn_ccl_labels_f64": [_P, _P, _I64, _I64, _I64, _RIGP, _D, _I64, _P, _P],
    "sn_ccl_labels_ws_f64": [_P, _P, _I64, _I64, _I64, _RIGP, _D, _I64, _P, _P, ctypes.c_size_t,
                             _P],
    "sn_adaptive_workspace_bytes": [_I64, _I64, _I64, ctypes.POINTER(ctypes.c_size_t)],
    "sn_adaptive_points": [_P, _P, _I64, _I64, _I64, _RIGP, _I32, _P, _P, _I32, _I32, _D, _P, _P,
                           _P, ctypes.c_size_t, _P],
    "sn_eval_workspace_bytes": [_I64, _I64, _I64, ctypes.POINTER(ctypes.c_size_t)],
    "sn_angular_error": [_P, _P, _I32, _P, _P, _P, _I64, _I64, _I64, _P, _P, _P, ctypes.c_size_t, _P],
    "sn_error_stats": [_P, _P, _I64, _I64, _I64, _P, _P, ctypes.c_size_t, _P],
    "sn_angular_error_f64": [_P, _P, _I32, _P, _P, _P, _I64, _I64, _I64, _P, _P, _P,
                             ctypes.c_size_t, _P],
    "sn_dequant_png16": [_P, _P, _I64, _I64, _I64, _D, _I32, _P, _P, _P],
    "sn_decode_pfm": [_P, _P, _I64, _I64, _I64, _I32, _I32, _P, _P],
    "sn_oriented_points_png16": [_P, _P, _I64, _I64, _I64, _D, _I32, _RIGP, _P, _I32, _P, _P,
                                 _P],
    "sn_cloud_workspace_bytes": [_I64, _I64, _I64, ctypes.POINTER(ctypes.c_size_t)],
    "sn_compact_cloud": [_P, _P, _P, _I64, _I64, _I64, _P, _I64, _P, _P, ctypes.c_size_t, _P],
    "sn_cloud_count": [_P, _P, _I64, _I64, _I64, _P, _P, ctypes.c_size_t, _P],
    "sn_cloud_scatter": [_P, _P, _P, _I64, _I64, _I64, _P, _I64, _P, ctypes.c_size_t, _P],
    "sn_pipeline": [_P, _P, _I64, _I64, _I64, _RIGP, _P, _I32, _D, _P, _P, _P, _P],
    "sn_pipeline_ws": [_P, _P, _I64, _I64, _I64, _RIGP, _P, _I32, _D, _P, _P, _P, _P,
                       ctypes.c_size_t, _P],
    "sn_ccl_from_bits_ws": [_P, _P, _I64, _I64, _I64, _I64, _P, _P, ctypes.c_size_t, _P],
    "sn_oriented_points_host": [_P, _P, _I64, _I64, _I64, _RIGP, _P, _I32, _P, _P],
    "sn_pipeline_host": [_P, _P, _I64, _I64, _I64, _RIGP, _P, _I32, _D, _P, _P, _P],
    "sn_pipeline_host_f64": [_P, _P, _I64, _I64, _I64, _RIGP, _P, _I32, _D, _P, _P, _P],
    "sn_oriented_points_host_f64": [_P, _P, _I64, _I64, _I64, _RIGP, _P, _I32, _P, _P],
    "sn_affine": [_P, _P, _I64, _I64, _I64, _P, _I32, _P, _P, _P, _P],
    "sn_affine_f64": [_P, _P, _I64, _I64, _I64, _P, _I32, _P, _P, _P, _P],
    "sn_passable": [_P, _P, _I64, _I64, _I64, _RIGP, _D, _P, _P, _P],
    "sn_ccl_labels": [_P, _P, _I64, _I64, _I64, _RIGP, _D, _I64, _P, _P],
    "sn_ccl_from_passable": [_P, _P, _I64, _I64, _I64, _I64, _P, _P],
    "sn_ccl_workspace_bytes": [_I64, _I64, _I64, ctypes.POINTER(ctypes.c_size_t)],
    "sn_ccl_labels_ws": [_P, _P, _I64, _I64, _I64, _RIGP, _D, _I64, _P, _P, ctypes.c_size_t, _P],
    "sn_ccl_from_passable_ws": [_P, _P, _I64, _I64, _I64, _I64, _P, _P, ctypes.c_size_t, _P],
    "sn_seam_merge_host": [_P, _I32, _I64, _P, _P, _P],
    "sn_depth_map": [_P, _P, _I64, _RIGP, _P, _P],
    "sn_depth_map_f64": [_P, _P, _I64, _RIGP, _P, _P],
    "sn_triangulate_f64": [_P, _P, _P, _P, _I64, _RIGP, _P, _P, _P, _P],
    "sn_triangulate_grid": [_P, _P, _I64, _I64, _I64, _RIGP, _P, _P],
    "sn_triangulate_grid_f64": [_P, _P, _I64, _I64, _I64, _RIGP, _P, _P],
    "sn_depth_laplacian_f64": [_P, _P, _P, _I64, _I64, _I64, _P, _P, _P],
    "sn_relabel": [_P, _P, _I64, _I64, _P, _P, _P, _I32, _P, _P],
    "sn_seam_merge": [_P, _P, _I32, _I64, _P, _I64, _P],
    "sn_relabel_table": [_P, _P, _I64, _P, _I64, _P],
}
_RESTYPES = {"sn_last_error": ctypes.c_char_p}

_lib = None
_lock = threading.Lock()
_plans: dict[int, ctypes.c_void_p] = {}


def load():
    """Load (once) and return the ctypes library; raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = os.environ.get("SN_B200_LIB", str(LIB_PATH))
        if not Path(path).exists():
            raise NativeLibraryError(
                f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback for the stereonorm-b200 hot path)")
        try:
            lib = ctypes.CDLL(path)
        except OSError as exc:  # pragma: no cover - environment dependent
            raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, ctypes.c_int)
        _lib = lib
        return lib


def last_error() -> str:
    return load().sn_last_error().decode("utf-8", "replace")


def check(rc: int, what: str = "") -> None:
    if rc == SN_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == SN_EINVAL:
        raise ValueError(msg)
    if rc == SN_EDEGENERATE:
        raise DegenerateSupportError(msg)
    raise RuntimeError(msg)


def plan(device: int):
    """Per-device plan handle (created lazily, lives for the process)."""
    p = _plans.get(device)
    if p is not None:
        return p
    with _lock:
        p = _plans.get(device)
        if p is None:
            h = ctypes.c_void_p()
            rc = load().sn_plan_create(int(device), ctypes.byref(h))
            check(rc, "sn_plan_create")
            _plans[device] = h
            p = h
    return p


def ccl_workspace_bytes(B: int, H: int, W: int) -> int:
    n = ctypes.c_size_t(0)
    check(load().sn_ccl_workspace_bytes(int(B), int(H), int(W), ctypes.byref(n)),
          "sn_ccl_workspace_bytes")
    return int(n.value)


def rig_struct(rig) -> SnRig:
    return SnRig(float(rig.fx), float(rig.fy), float(rig.u0), float(rig.v0), float(rig.baseline))


def offsets_array(offsets) -> np.ndarray:
    off = np.ascontiguousarray(np.asarray(offsets, dtype=np.int32).reshape(-1, 2))
    return off


def kernel_moments(offsets) -> SnMoments:
    off = offsets_array(offsets)
    m = SnMoments()
    rc = load().sn_kernel_moments(off.ctypes.data if off.size else None, int(len(off)),
                                  ctypes.byref(m))
    check(rc, "build_kernels")
    return m
