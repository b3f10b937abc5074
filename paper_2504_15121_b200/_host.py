"""numpy <-> device staging for the reference-facing host API."""

from __future__ import annotations

import numpy as np
import torch


def resolve_threads(threads) -> int:
    """Reference threading knob (parallel.py:35-40): validated for drop-in
    compatibility; the GPU path's result does not depend on it."""
    if threads is None:
        return 1
    if int(threads) < 1:
        raise ValueError("thread count must be >= 1")
    return int(threads)


def current_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("stereonorm-b200 needs a CUDA device (no CPU fallback exists)")
    return torch.device("cuda", torch.cuda.current_device())


def to_device(values: np.ndarray, dtype=torch.float64) -> torch.Tensor:
    arr = np.ascontiguousarray(values)
    return torch.from_numpy(arr).to(device=current_device(), dtype=dtype, non_blocking=False)


def stream_ptr(dev: torch.device):
    import ctypes
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()
