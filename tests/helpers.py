import numpy as np


def rig_of(arr):
    from paper_2504_15121_b200 import StereoRig
    fx, fy, u0, v0, b = (float(v) for v in arr)
    return StereoRig(fx, fy, u0, v0, b)


def orig_of(arr):
    from oracle.stereonorm_oracle import Rig
    fx, fy, u0, v0, b = (float(v) for v in arr)
    return Rig(fx, fy, u0, v0, b)


def max_angle_deg(a, b):
    """Unsigned angle between unit-ish vectors (rows), degrees."""
    if len(a) == 0:
        return 0.0
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    a = a / np.linalg.norm(a, axis=-1, keepdims=True)
    b = b / np.linalg.norm(b, axis=-1, keepdims=True)
    # sine form is accurate for tiny angles
    s = np.linalg.norm(np.cross(a, b), axis=-1)
    c = np.abs(np.sum(a * b, axis=-1))
    return float(np.degrees(np.arctan2(s, c)).max())


def max_rel(a, b, floor=0.0):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if a.size == 0:
        return 0.0
    den = np.maximum(np.abs(b), floor)
    with np.errstate(invalid="ignore", divide="ignore"):
        r = np.abs(a - b) / den
    return float(np.nanmax(np.where(den > 0, r, np.abs(a - b))))


def max_point_rel(a, b):
    """max |a - b| / |b| over points (rows); the 1e-5 bar of the north star."""
    a = np.asarray(a, np.float64).reshape(-1, 3)
    b = np.asarray(b, np.float64).reshape(-1, 3)
    if len(a) == 0:
        return 0.0
    return float((np.linalg.norm(a - b, axis=-1) / np.linalg.norm(b, axis=-1)).max())
