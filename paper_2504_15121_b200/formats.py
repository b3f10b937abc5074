"""Oriented PLY output of the dense cloud.

Byte-compatible with the reference writer ``write_ply_oriented``
(formats.py:167-211): header ``ply`` / ``format binary_little_endian 1.0``
(or ``ascii 1.0``) / ``element vertex N`` / six ``property float`` lines
(x y z nx ny nz) / ``end_header``, then little-endian float32 rows in source
(raster) order.  The device compaction (``device.compact_cloud``) already
produces the binary body, so ``ply_from_vertices`` only prepends the header.
"""

from __future__ import annotations

import numpy as np

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
