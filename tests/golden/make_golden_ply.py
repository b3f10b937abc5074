"""Golden PLY bytes from the REFERENCE writer (formats.py:170-185).

Run in the build container (reads /root/reference):

    python tests/golden/make_golden_ply.py

Stores a small vertex set (with the signed zeros, tiny/huge magnitudes and
an empty cloud) and the reference's binary and ASCII encodings.
"""

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from stereonorm import formats  # noqa: E402

OUT = Path(__file__).resolve().parent
rng = np.random.default_rng(21)
pts = rng.normal(0, 50, (37, 3)).astype(np.float32)
nrm = rng.normal(0, 1, (37, 3))
nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
nrm = nrm.astype(np.float32)
pts[0] = [0.0, -0.0, 1e-30]
pts[1] = [3.4e38, -1.2e-38, 7.0]
arrays = {"points": pts, "normals": nrm}
for binary in (True, False):
    tag = "bin" if binary else "ascii"
    arrays[f"ply_{tag}"] = np.frombuffer(formats.write_ply_oriented(pts, nrm, binary), np.uint8)
    arrays[f"empty_{tag}"] = np.frombuffer(
        formats.write_ply_oriented(np.zeros((0, 3)), np.zeros((0, 3)), binary), np.uint8)
np.savez_compressed(OUT / "ply_cases.npz", **arrays)
print("wrote", OUT / "ply_cases.npz")
