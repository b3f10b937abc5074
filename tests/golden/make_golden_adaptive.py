"""Golden vectors for the adaptive star-fill path, from the REFERENCE package
(adaptive.py:177-268 estimate_normals_adaptive; StarConfig adaptive.py:32-57).

Run in the build container (reads /root/reference):

    python tests/golden/make_golden_adaptive.py

Inputs are fp32-rounded disparities of small scene crops (street, sphere)
with PCG64 noise and holes; configs cover both stop rules, shared_range,
3..16 directions and 1..30 steps.
"""

import json
import sys
from pathlib import Path

import numpy as np
from scipy import ndimage

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import stereonorm as sn  # noqa: E402
from paper_2504_15121_b200 import scenes  # noqa: E402  (host-side scene synthesis only)

OUT = Path(__file__).resolve().parent


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def street(w, h, sigma, seed, holes=0.0):
    sc = scenes.street_scene(w, h, fx=float(w))
    d = scenes.add_gaussian_noise(scenes.raycast(sc)[0], sigma, seed)
    if holes:
        m = ndimage.binary_dilation(np.random.default_rng(seed + 100).random(d.shape) < holes,
                                    iterations=2)
        d[m] = np.nan
    return f32(d), sc.rig


def sphere(w, h, sigma, seed):
    sp = scenes.sphere_scene(w, h, fx=float(w))
    return f32(scenes.add_gaussian_noise(scenes.raycast(sp)[0], sigma, seed)), sp.rig


CASES = [
    ("street_cd_d8_s10", street(192, 112, 0.2, 1), dict(stop="cd", threshold=0.1)),
    ("street_st_d8_s10", street(192, 112, 0.05, 2), dict(stop="st", threshold=1.0)),
    ("street_cd_shared", street(160, 96, 0.2, 3),
     dict(stop="cd", threshold=0.2, shared_range=True)),
    ("street_cd_holes", street(200, 120, 0.2, 4, holes=0.004), dict(stop="cd", threshold=0.1)),
    ("street_st_holes", street(200, 120, 0.05, 5, holes=0.004), dict(stop="st", threshold=2.0)),
    ("sphere_cd_d16_s5", sphere(128, 128, 0.2, 7),
     dict(stop="cd", threshold=0.05, directions=16, max_steps=5)),
    ("sphere_st_d3_s2", sphere(96, 96, 0.2, 8),
     dict(stop="st", threshold=0.5, directions=3, max_steps=2)),
    ("sphere_cd_d5_s30", sphere(96, 80, 0.2, 9),
     dict(stop="cd", threshold=0.3, directions=5, max_steps=30)),
    ("street_cd_s1", street(64, 48, 0.2, 10), dict(stop="cd", threshold=0.1, max_steps=1)),
    ("tiny", (f32(np.full((3, 4), 20.0)), sn.StereoRig(100.0, 100.0, 1.5, 1.0, 0.2)),
     dict(stop="cd", threshold=0.1)),
]


def main():
    arrays, index = {}, []
    for name, (d, rig), cfg in CASES:
        field = sn.ScalarField.from_array(d)
        nf = sn.estimate_normals_adaptive(field, rig, sn.StarConfig(**cfg))
        arrays[f"{name}__d"] = d
        arrays[f"{name}__rig"] = np.array([rig.fx, rig.fy, rig.u0, rig.v0, rig.baseline])
        arrays[f"{name}__normals"] = nf.vectors
        arrays[f"{name}__nmask"] = nf.mask
        index.append({"name": name, "config": cfg, "valid": float(nf.mask.mean())})
    arrays["names"] = np.array([c["name"] for c in index])
    arrays["configs"] = np.array([json.dumps(c["config"]) for c in index])
    np.savez_compressed(OUT / "adaptive_cases.npz", **arrays)
    for c in index:
        print(f"{c['name']:20s} valid {c['valid']:.3f}  {c['config']}")


if __name__ == "__main__":
    main()
