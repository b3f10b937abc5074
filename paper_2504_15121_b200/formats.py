"""Readers and writers either side of the hot path.

Inputs (f3): PFM and 16-bit PNG disparity files.  The container is parsed on
the host -- the PFM header (formats.py:55-81) here, the PNG zlib stream by
PIL as in the reference (formats.py:133-150) -- and the per-sample work runs
on the device (``device.decode_pfm`` / ``device.dequant_png16``) after one
copy of the raw payload.  ``read_pfm`` / ``read_disparity_png16`` keep the
reference's signatures, ScalarField results and FormatError behaviour; the
``*_device`` variants return the CUDA tensor the fused pass consumes.

Output (f2): oriented PLY.

Byte-compatible with the reference writer ``write_ply_oriented``
(formats.py:167-211): header ``ply`` / ``format binary_little_endian 1.0``
(or ``ascii 1.0``) / ``element vertex N`` / six ``property float`` lines
(x y z nx ny nz) / ``end_header``, then little-endian float32 rows in source
(raster) order.  The device compaction (``device.compact_cloud``) already
produces the binary body, so ``ply_from_vertices`` only prepends the header.
"""

from __future__ import annotations

import io
import re

import numpy as np
import torch

from .fields import NormalField, ScalarField


class FormatError(Exception):
    """Malformed file content; ``offset`` is the parse position if known
    (formats.py:40-47)."""

    def __init__(self, message: str, offset: int | None = None):
        if offset is not None:
            message = f"{message} (at byte {offset})"
        super().__init__(message)
        self.offset = offset


# --------------------------------------------------------------------------
# PFM (formats.py:55-113)

# one header token: optional ASCII whitespace (bytes.isspace), then a run of
# non-whitespace bytes
_TOKEN = re.compile(rb"[ \t\n\r\x0b\x0c]*([^ \t\n\r\x0b\x0c]+)")
_SPACE = b" \t\n\r\x0b\x0c"


def _pfm_header(data: bytes):
    """(magic, width, height, scale, payload offset) of a PFM header: four
    whitespace-separated tokens and exactly one whitespace byte before the
    payload.  Error messages and offsets are the reference's
    (formats.py:55-81)."""
    fields, end = [], 0
    for _ in range(4):
        m = _TOKEN.match(data, end)
        if m is None:  # only whitespace (or nothing) left
            raise FormatError("truncated PFM header", offset=len(data))
        fields.append(m.group(1))
        end = m.end()
    if end == len(data) or data[end] not in _SPACE:
        raise FormatError("missing whitespace after PFM scale", offset=end)
    magic, w_tok, h_tok, s_tok = fields
    if magic != b"Pf" and magic != b"PF":
        raise FormatError(f"bad PFM magic {magic!r}", offset=0)
    try:
        dims = (int(w_tok), int(h_tok))
        scale = float(s_tok)
    except ValueError as exc:
        raise FormatError(f"bad PFM header field: {exc}") from None
    if min(dims) <= 0:
        raise FormatError(f"bad PFM dimensions {dims[0]}x{dims[1]}")
    if scale == 0.0:
        raise FormatError("PFM scale must be nonzero")
    return magic, dims[0], dims[1], scale, end + 1


def read_pfm_device(data: bytes, magic: bytes = b"Pf", device=None) -> torch.Tensor:
    """Decode a PFM on the device: float32 ``[H, W]`` (``[H, W, 3]`` for
    ``PF``), top row first, NaN/inf samples kept (they mark invalid pixels)."""
    magic_, width, height, scale, pos = _pfm_header(data)
    if magic_ != magic:
        kind = "grayscale 'Pf'" if magic == b"Pf" else "3-channel 'PF'"
        raise FormatError(f"expected {kind} PFM, got {magic_.decode()!r}", offset=0)
    ch = 3 if magic == b"PF" else 1
    need = width * height * ch * 4
    have = len(data) - pos
    if have < need:
        raise FormatError(f"truncated PFM payload: need {need} bytes, have {have}",
                          offset=pos + have)
    from . import device as _dev
    from ._host import current_device
    dev = torch.device(device) if device is not None else current_device()
    host = torch.frombuffer(bytearray(data[pos:pos + need]), dtype=torch.uint8)
    out = _dev.decode_pfm(host.to(dev), height, width, ch, big_endian=scale > 0)
    return out[0]


def read_pfm(data: bytes) -> ScalarField:
    """Grayscale PFM to a scalar field; non-finite samples become invalid
    (formats.py:105-108)."""
    return ScalarField.from_array(read_pfm_device(data, b"Pf").double().cpu().numpy())


def read_pfm_normals(data: bytes) -> NormalField:
    """3-channel PFM to a normal field (formats.py:118-121)."""
    return NormalField.from_array(read_pfm_device(data, b"PF").double().cpu().numpy())


def _pfm_bytes(magic: str, grid: np.ndarray) -> bytes:
    """Little-endian PFM (negative scale), rows bottom-up as float32."""
    h, w = grid.shape[:2]
    body = np.ascontiguousarray(np.flip(grid, axis=0), dtype="<f4")
    return b"".join((f"{magic}\n{w} {h}\n-1.0\n".encode("ascii"), body.tobytes()))


def write_pfm(field: ScalarField) -> bytes:
    """Grayscale PFM, invalid pixels as NaN (formats.py:111-115)."""
    return _pfm_bytes("Pf", field.values)


def write_pfm_normals(field: NormalField) -> bytes:
    """3-channel PFM (formats.py:124-127)."""
    return _pfm_bytes("PF", field.vectors)


# --------------------------------------------------------------------------
# 16-bit disparity PNG (formats.py:130-162)

def _png16_samples(data: bytes) -> np.ndarray:
    """The PNG container (zlib + filters) decoded by PIL, as the reference
    does; returns the raw 16-bit samples.  Rejections carry the reference's
    messages (formats.py:135-146)."""
    from PIL import Image
    try:
        with Image.open(io.BytesIO(data)) as img:
            img.load()
            kind, mode, raw = img.format, img.mode, np.asarray(img)
    except Exception as exc:
        raise FormatError(f"not a decodable PNG: {exc}") from None
    problem = (f"expected PNG, got {kind}" if kind != "PNG" else
               f"expected 16-bit single-channel PNG, got mode {mode!r}"
               if mode not in ("I;16", "I") else None)
    if problem:
        raise FormatError(problem)
    ok = raw.ndim == 2 and raw.size > 0 and 0 <= int(raw.min()) and int(raw.max()) <= 0xFFFF
    if not ok:
        raise FormatError("PNG samples out of 16-bit range")
    return raw.astype(np.uint16)


def read_disparity_png16_device(data: bytes, scale: float = 256.0, invalid_value: int = 0,
                                dtype=torch.float32, device=None) -> torch.Tensor:
    """Dequantised disparity ``[H, W]`` on the device (NaN where raw ==
    invalid_value); float64 is the reference's value exactly."""
    from . import device as _dev
    from ._host import current_device
    dev = torch.device(device) if device is not None else current_device()
    raw = torch.from_numpy(_png16_samples(data)).to(dev)
    inv = int(invalid_value)
    return _dev.dequant_png16(raw, scale, inv if 0 <= inv <= 0xFFFF else None, dtype=dtype)[0]


def read_png16_raw_device(data: bytes, device=None) -> torch.Tensor:
    """The undecoded 16-bit samples on the device, for
    ``device.oriented_points_png16`` (2 B/px into the fused pass)."""
    from ._host import current_device
    dev = torch.device(device) if device is not None else current_device()
    return torch.from_numpy(_png16_samples(data)).to(dev)


def read_disparity_png16(data: bytes, scale: float = 256.0,
                         invalid_value: int = 0) -> ScalarField:
    """Quantised disparity: d = (raw - 1) / scale, raw == invalid_value masked
    (formats.py:133-150)."""
    raw = _png16_samples(data)
    mask = raw.astype(np.int64) != invalid_value
    d = read_disparity_png16_device(data, scale, invalid_value, dtype=torch.float64)
    return ScalarField(d.cpu().numpy(), mask)


def write_disparity_png16(field: ScalarField, scale: float = 256.0,
                          invalid_value: int = 0) -> bytes:
    """Inverse of read_disparity_png16; valid raws clamp to [1, 65535]
    (formats.py:153-162)."""
    from PIL import Image
    # quantise the valid samples only (round half to even, then clamp into the
    # raw range 1 .. 65535); every other pixel carries the invalid raw value
    q = np.full(field.values.shape, invalid_value, dtype=np.uint16)
    valid = np.asarray(field.mask, dtype=bool)
    q[valid] = np.clip(np.rint(field.values[valid] * float(scale) + 1.0), 1.0, 65535.0)
    out = io.BytesIO()
    Image.fromarray(q).save(out, format="PNG")
    return out.getvalue()


# --------------------------------------------------------------------------
# PLY

PLY_PROPS = ("x", "y", "z", "nx", "ny", "nz")


def _header(n: int, binary: bool) -> bytes:
    fmt = "binary_little_endian" if binary else "ascii"
    lines = ["ply", f"format {fmt} 1.0", f"element vertex {n}"]
    lines += [f"property float {p}" for p in PLY_PROPS]
    lines.append("end_header")
    return ("\n".join(lines) + "\n").encode("ascii")


def ply_from_vertices(vertices, binary: bool = True) -> bytes:
    """PLY bytes of ``[N, 6]`` float32 vertices (x, y, z, nx, ny, nz)."""
    rows = np.ascontiguousarray(np.asarray(vertices, dtype="<f4").reshape(-1, 6))
    if binary:
        return _header(len(rows), True) + rows.tobytes()
    body = "\n".join(" ".join(f"{v:.9g}" for v in row) for row in rows)
    return _header(len(rows), False) + (body + "\n" if len(rows) else "").encode("ascii")


def write_ply_oriented(points, normals, binary: bool = True) -> bytes:
    """Reference signature (formats.py:170): points and unit normals (N, 3)."""
    pts = np.asarray(points, dtype=np.float32).reshape(-1, 3)
    nrm = np.asarray(normals, dtype=np.float32).reshape(-1, 3)
    if len(pts) != len(nrm):
        raise ValueError(f"point/normal count mismatch: {len(pts)} vs {len(nrm)}")
    return ply_from_vertices(np.hstack([pts, nrm]), binary)
