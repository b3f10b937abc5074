"""Host-side helpers of the drop-in API against the REFERENCE (stereonorm
0.1.0): format_kernel_dump text, estimate_affine_direct values and the PFM
writers' bytes.  Run in the build container (reads /root/reference):

    python tests/golden/make_golden_host.py
"""

import base64
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import stereonorm as sn  # noqa: E402

OUT = Path(__file__).resolve().parent

SPECS = {
    "sq3": sn.KernelSpec.square(3), "sq5": sn.KernelSpec.square(5), "sq9": sn.KernelSpec.square(9),
    "cross4": sn.KernelSpec(np.array([[1, 0], [-1, 0], [0, 1], [0, -1]])),
    "sparse5": sn.KernelSpec(np.array([[0, 0], [2, 1], [1, 2], [-2, -1], [3, -2]])),
    "asym6": sn.KernelSpec(np.array([[0, 0], [1, 0], [2, 0], [0, 1], [0, 2], [1, 1]])),
}


def main():
    rng = np.random.default_rng(5)
    d = 20.0 + np.cumsum(rng.normal(0, 0.3, (40, 50)), axis=1) + rng.normal(0, 0.05, (40, 50))
    d[10:13, 20:24] = np.nan
    d[0, 0] = np.inf
    field = sn.ScalarField.from_array(d)
    out = {"dumps": {k: sn.format_kernel_dump(sn.build_kernels(s)) for k, s in SPECS.items()},
           "disparity": [[None if not np.isfinite(x) else float(x) for x in row] for row in d],
           "direct": []}
    pix = [(0, 0), (1, 1), (49, 39), (22, 11), (21, 9), (25, 14), (5, 30)] + \
          [(int(rng.integers(0, 50)), int(rng.integers(0, 40))) for _ in range(30)]
    for name, spec in SPECS.items():
        for u, v in pix:
            a1, a2 = sn.estimate_affine_direct(field, (u, v), spec)
            out["direct"].append({"spec": name, "pixel": [u, v], "a1": a1, "a2": a2})
    nf = sn.NormalField.from_array(rng.normal(size=(7, 9, 3)))
    out["pfm"] = base64.b64encode(sn.formats.write_pfm(field)).decode()
    out["pfm_normals"] = base64.b64encode(sn.formats.write_pfm_normals(nf)).decode()
    out["normals"] = nf.vectors.tolist()
    (OUT / "host_cases.json").write_text(json.dumps(out))


if __name__ == "__main__":
    main()
