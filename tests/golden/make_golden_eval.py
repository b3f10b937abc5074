"""Golden vectors for the accuracy evaluation, from the REFERENCE package
(evaluation.py:34-73: angular_error_map, summarize).

Run in the build container (reads /root/reference):

    python tests/golden/make_golden_eval.py

Cases: the shipped sphere scene (reduced to 256x256) with the reference's own
ground-truth normals, estimated by the reference's fixed 9x9 and adaptive CD
estimators from a noisy disparity, with and without an extra mask; an
odd-count case for the lower median.
"""

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import stereonorm as sn  # noqa: E402
from stereonorm import evaluation, synth  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    rig = sn.StereoRig(256.0, 256.0, 127.5, 127.5, 0.3)
    scene = synth.SceneSpec(width=256, height=256, rig=rig,
                            primitives=[synth.Sphere((0.0, 0.0, 3.0), 1.4)])
    gt = synth.raycast(scene)
    noisy = synth.add_gaussian_noise(gt.disparity, 0.2, 7)
    d = np.where(noisy.mask, noisy.values, np.nan).astype(np.float32).astype(np.float64)
    field = sn.ScalarField.from_array(d)
    arrays = {"gt_n": gt.normals.vectors, "gt_m": gt.normals.mask}
    names = []
    ests = {
        "fixed9": sn.estimate_normals_fixed(field, rig, 9),
        "adaptive_cd": sn.estimate_normals_adaptive(field, rig, sn.StarConfig()),
    }
    ring = np.zeros((256, 256), bool)
    ring[60:200, 40:220] = True
    for name, est in ests.items():
        for mtag, mask in (("all", None), ("ring", ring)):
            err = evaluation.angular_error_map(est, gt.normals, mask)
            st = evaluation.summarize(err)
            tag = f"{name}_{mtag}"
            names.append(tag)
            arrays[f"{tag}__est_n"] = est.vectors
            arrays[f"{tag}__est_m"] = est.mask
            arrays[f"{tag}__mask"] = mask if mask is not None else np.ones((256, 256), bool)
            arrays[f"{tag}__err"] = np.where(err.mask, err.values, np.nan)
            arrays[f"{tag}__stats"] = np.array([st.avg, st.min, st.max, st.median, st.std,
                                                st.valid_count], dtype=np.float64)
            print(tag, st)
    arrays["names"] = np.array(names)
    np.savez_compressed(OUT / "eval_cases.npz", **arrays)


if __name__ == "__main__":
    main()
