"""Golden vectors on the reference's OWN float64 inputs (no fp32 rounding),
produced by the REFERENCE package (stereonorm 0.1.0).

Run in the build container (reads /root/reference):

    python tests/golden/make_golden_f64.py

Covers the rows whose decisions must be bit-exact on float64 disparities:
the ST predicate and edge values (geometry.py:169-172 depth_field,
adaptive.py:80-97 depth_laplacian, the ST test adaptive.py:130-132), the
component labels of that passable set (scipy.ndimage.label, 8-connectivity,
min-raster-index relabel: SURVEY.md §8 A10), the adaptive star-fill masks
(adaptive.py:177-268), star_trace supports (adaptive.py:100-143) and the
element-wise geometry (disparity_to_depth, triangulate, triangulate_grid,
geometry.py:39-89).

Large inputs are not stored: they are regenerated in the tests from the
seeds with ``paper_2504_15121_b200.scenes`` (which reproduces the reference's
synth.raycast / add_gaussian_noise bit for bit, tests/test_host_cpu.py) and
checked against the SHA-256 of the float64 bytes recorded here.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np
from scipy import ndimage

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import stereonorm as sn  # noqa: E402
from paper_2504_15121_b200 import scenes  # noqa: E402  (input synthesis only)

OUT = Path(__file__).resolve().parent
THRESHOLDS = (0.05, 0.2, 1.0)


def street_input(w, h, sigma, seed, holes=False):
    """SURVEY.md §8(d) C3/C4 recipe at w x h (fx = w): street raycast +
    N(0, sigma) PCG64(seed) noise; C4 holes = binary_dilation(rng(1000 +
    seed).random < 0.002, iterations=3)."""
    sc = scenes.street_scene(w, h)
    d = scenes.add_gaussian_noise(scenes.raycast(sc)[0], sigma, seed)
    if holes:
        m = ndimage.binary_dilation(np.random.default_rng(1000 + seed).random(d.shape) < 0.002,
                                    iterations=3)
        d = np.where(m, np.nan, d)
    return d, sc.rig


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def ref_rig(r):
    return sn.StereoRig(r.fx, r.fy, r.u0, r.v0, r.baseline)


def labels_of(p):
    lab, n = ndimage.label(p, structure=np.ones((3, 3), dtype=int))
    out = np.full(p.shape, -1, dtype=np.int64)
    if n:
        flat = lab.ravel()
        idx = np.flatnonzero(flat)
        first = np.full(n + 1, np.iinfo(np.int64).max)
        np.minimum.at(first, flat[idx], idx)
        out.ravel()[idx] = first[flat[idx]]
    return out.astype(np.int32)


def passable_of(d, rig, t):
    field = sn.ScalarField.from_array(d)
    e = sn.depth_laplacian(sn.depth_field(field, rig))
    with np.errstate(invalid="ignore"):
        return e, e.mask & (e.values <= t)


# inputs regenerated from seeds in the tests: (name, w, h, sigma, seed, holes)
FRAMES = [
    ("street_1024_s02_seed3", 1024, 512, 0.2, 3, False),
    ("street_512_s10_holes_seed5", 512, 256, 1.0, 5, True),
    ("street_512_s02_seed11", 512, 256, 0.2, 11, False),
]

ADAPTIVE = [
    ("st_t1_s005", (192, 112, 0.05, 2, False), dict(stop="st", threshold=1.0)),
    ("st_t02_s02", (192, 112, 0.2, 6, False), dict(stop="st", threshold=0.2)),
    ("st_holes", (200, 120, 1.0, 4, True), dict(stop="st", threshold=2.0)),
    ("cd_t01", (192, 112, 0.2, 1, False), dict(stop="cd", threshold=0.1)),
    ("cd_shared", (160, 96, 0.2, 3, False), dict(stop="cd", threshold=0.2, shared_range=True)),
    ("cd_holes_d16", (200, 120, 1.0, 7, True),
     dict(stop="cd", threshold=0.05, directions=16, max_steps=5)),
]


def main():
    arrays, meta = {}, {"frames": [], "adaptive": [], "flips": {}}
    for name, w, h, sigma, seed, holes in FRAMES:
        d, r = street_input(w, h, sigma, seed, holes)
        rig = ref_rig(r)
        entry = {"name": name, "w": w, "h": h, "sigma": sigma, "seed": seed, "holes": holes,
                 "sha256": sha(d)}
        small = w * h <= 512 * 256
        for t in THRESHOLDS:
            e, p = passable_of(d, rig, t)
            arrays[f"{name}__pass_{t}"] = np.packbits(p, axis=None)
            arrays[f"{name}__labels_{t}"] = labels_of(p)
            if small and t == THRESHOLDS[0]:
                arrays[f"{name}__edges"] = e.values
            # what rounding the input to fp32 would have changed
            _, p32 = passable_of(d.astype(np.float32).astype(np.float64), rig, t)
            meta["flips"][f"{name}@{t}"] = int((p32 != p).sum())
        # thresholds equal to edge values of the frame: exact ties e == t
        # (passable, since the test is e <= t) that an fp32 input would move
        e, _ = passable_of(d, rig, 1.0)
        ev = np.sort(e.values[e.mask])
        ties = [float(ev[int(q * (len(ev) - 1))]) for q in (0.1, 0.3, 0.5, 0.7, 0.9)]
        entry["ties"] = ties
        for i, t in enumerate(ties):
            _, p = passable_of(d, rig, t)
            arrays[f"{name}__tie_{i}"] = np.packbits(p, axis=None)
            _, p32 = passable_of(d.astype(np.float32).astype(np.float64), rig, t)
            meta["flips"][f"{name}@tie{i}"] = int((p32 != p).sum())
        arrays[f"{name}__tie_labels"] = labels_of(passable_of(d, rig, ties[2])[1])
        meta["frames"].append(entry)

    for name, (w, h, sigma, seed, holes), cfg in ADAPTIVE:
        d, r = street_input(w, h, sigma, seed, holes)
        rig = ref_rig(r)
        conf = sn.StarConfig(**cfg)
        field = sn.ScalarField.from_array(d)
        nf = sn.estimate_normals_adaptive(field, rig, conf)
        arrays[f"{name}__normals"] = nf.vectors.astype(np.float32)
        arrays[f"{name}__nmask"] = nf.mask
        # star_trace supports of a few pixels (adaptive.py:100-143)
        depth = sn.depth_field(field, rig)
        edges = sn.depth_laplacian(depth) if conf.stop == "st" else None
        rng = np.random.default_rng(seed)
        pix = [(int(rng.integers(0, w)), int(rng.integers(0, h))) for _ in range(24)]
        pix += [(0, 0), (w - 1, h - 1), (w // 2, 0), (3, h // 2)]
        traces = []
        for u, v in pix:
            off = sn.star_trace((u, v), depth, edges, conf)
            a1, a2 = sn.estimate_affine_adaptive(field, depth, edges, (u, v), conf)
            traces.append({"pixel": [u, v], "offsets": off.tolist(), "a1": a1, "a2": a2})
        meta["adaptive"].append({"name": name, "w": w, "h": h, "sigma": sigma, "seed": seed,
                                 "holes": holes, "config": cfg, "sha256": sha(d),
                                 "traces": traces})

    # element-wise geometry on special values (geometry.py:39-89)
    rig = sn.StereoRig(fx=1234.5, fy=1200.25, u0=611.3, v0=187.9, baseline=0.537)
    specials = np.array([np.nan, np.inf, -np.inf, 0.0, -0.0, -3.5, 5e-324, 1e-310, 1e-300,
                         1e-30, 0.1, 1.0, 3.141592653589793, 77.25, 1e30, 1e300,
                         np.finfo(np.float64).max, 2.0 ** -1074 * 3])
    rng = np.random.default_rng(42)
    dvals = np.concatenate([specials, rng.uniform(0.5, 300.0, 200), rng.normal(0, 50, 50)])
    arrays["geom__d"] = dvals
    arrays["geom__rig"] = np.array([rig.fx, rig.fy, rig.u0, rig.v0, rig.baseline])
    arrays["geom__depth"] = sn.disparity_to_depth(dvals, rig)
    u = rng.uniform(-50, 1300, dvals.size)
    v = rng.uniform(-20, 400, dvals.size)
    arrays["geom__u"], arrays["geom__v"] = u, v
    x, y, z = sn.triangulate(u, v, dvals, rig)
    arrays["geom__x"], arrays["geom__y"], arrays["geom__z"] = x, y, z
    # broadcasting: a row of u against a column of d, scalar v
    ub, db = u[:7], dvals[:11, None]
    xb, yb, zb = sn.triangulate(ub, 42.0, db, rig)
    arrays["geom__bx"], arrays["geom__by"], arrays["geom__bz"] = xb, yb, zb
    # triangulate_grid / depth_field on a float64 frame with holes
    d, r = street_input(96, 64, 1.0, 9, True)
    d[5, 7], d[6, 7], d[7, 7] = -2.0, 0.0, 1e-310
    grid = d.copy()
    arrays["grid__d"] = grid
    rig_g = ref_rig(r)
    arrays["grid__rig"] = np.array([r.fx, r.fy, r.u0, r.v0, r.baseline])
    f = sn.ScalarField.from_array(grid)
    arrays["grid__points"] = sn.triangulate_grid(f, rig_g)
    df = sn.depth_field(f, rig_g)
    arrays["grid__depth"] = df.values
    arrays["grid__depth_mask"] = df.mask
    lap = sn.depth_laplacian(df)
    arrays["grid__lap"] = lap.values
    arrays["grid__lap_mask"] = lap.mask

    arrays["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(OUT / "f64_cases.npz", **arrays)
    print(json.dumps(meta["flips"], indent=1))
    print("adaptive:", [(a["name"], len(a["traces"])) for a in meta["adaptive"]])


if __name__ == "__main__":
    main()
