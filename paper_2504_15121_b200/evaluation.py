"""Angular-error maps and summary statistics on the GPU -- drop-in for the
reference's ``angular_error_map`` / ``summarize`` (evaluation.py:34-73,
SURVEY.md §8(f) f4).  The per-pixel angles, the reductions and the exact
lower median (radix select) run in csrc/sn_eval.cu; only the six numbers
come back to the host."""

from __future__ import annotations

from dataclasses import asdict, dataclass

import numpy as np

from .fields import NormalField, ScalarField

__all__ = ["ErrorStats", "angular_error_map", "summarize", "error_stats"]


@dataclass(frozen=True)
class ErrorStats:
    """Five-number summary of an error map, degrees, valid pixels only
    (evaluation.py:13-31)."""

    avg: float
    min: float
    max: float
    median: float
    std: float
    valid_count: int

    def as_dict(self) -> dict:
        return asdict(self)

    @classmethod
    def from_dict(cls, d: dict) -> "ErrorStats":
        return cls(avg=float(d["avg"]), min=float(d["min"]), max=float(d["max"]),
                   median=float(d["median"]), std=float(d["std"]),
                   valid_count=int(d["valid_count"]))


def _stats_of(row) -> ErrorStats:
    return ErrorStats(avg=float(row[0]), min=float(row[1]), max=float(row[2]),
                      median=float(row[3]), std=float(row[4]), valid_count=int(row[5]))


def _device_eval(est_vectors, gt: NormalField, mask, want_map):
    import torch
    from . import device
    from ._host import current_device

    dev = current_device()
    est = torch.from_numpy(np.ascontiguousarray(est_vectors, dtype=np.float64)).to(dev)
    g = torch.from_numpy(np.ascontiguousarray(gt.vectors, dtype=np.float64)).to(dev)
    gm = torch.from_numpy(np.ascontiguousarray(gt.mask)).to(dev)
    m = torch.from_numpy(np.ascontiguousarray(np.asarray(mask, dtype=bool))).to(dev) \
        if mask is not None else None
    return device.angular_error(est, g, gm, mask=m, want_map=want_map)


def angular_error_map(est: NormalField, gt: NormalField, mask=None) -> ScalarField:
    """Unsigned angle (degrees) between estimate and ground truth on jointly
    valid pixels (evaluation.py:34-55)."""
    if est.shape != gt.shape:
        raise ValueError(f"field sizes differ: {est.shape} vs {gt.shape}")
    vec = np.where(est.mask[..., None], est.vectors, np.nan)
    err, _ = _device_eval(vec, gt, mask, True)
    vals = err[0].cpu().numpy()
    return ScalarField(vals, np.isfinite(vals))


def error_stats(est: NormalField, gt: NormalField, mask=None) -> ErrorStats:
    """angular_error_map + summarize in one device pass (no map round trip)."""
    if est.shape != gt.shape:
        raise ValueError(f"field sizes differ: {est.shape} vs {gt.shape}")
    vec = np.where(est.mask[..., None], est.vectors, np.nan)
    _, stats = _device_eval(vec, gt, mask, False)
    row = stats[0].cpu().numpy()
    if not row[5] > 0:
        raise ValueError("cannot summarize an empty error map")
    return _stats_of(row)


def summarize(errors: ScalarField) -> ErrorStats:
    """Population statistics over the valid pixels of an error map
    (evaluation.py:58-73): lower median, std dividing by N."""
    import torch
    from . import device
    from ._host import current_device

    if not errors.mask.any():
        raise ValueError("cannot summarize an empty error map")
    vals = np.where(errors.mask, errors.values, np.nan)
    v = torch.from_numpy(np.ascontiguousarray(vals, dtype=np.float64)).to(current_device())
    return _stats_of(device.error_stats(v)[0].cpu().numpy())
