"""Generate golden vectors by running the REFERENCE package (stereonorm 0.1.0).

Run in the build container, where the read-only reference tree exists:

    python tests/golden/make_golden.py

It imports ``/root/reference/pkg/src/stereonorm`` and writes small ``.npz``
fixtures (inputs + the reference's own outputs) plus ``accuracy.json``.
Nothing on the GPU box reads the reference tree: the tests only load the
committed fixtures.

Case design follows the reference tests (pkg/tests/test_kernels.py:80-231,
test_geometry.py:29-77, test_adaptive.py:48-75) plus realistic scene crops
(street/sphere raycasts with PCG64 noise).  Disparities are
rounded to fp32 unless a case name ends in ``_f64``, so the fp32 device path
and the oracle see identical values.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
from scipy import ndimage

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
import stereonorm as sn  # noqa: E402


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def ramp(h, w, p, q, r):
    v, u = np.mgrid[0:h, 0:w].astype(float)
    return p + q * u + r * v


def street_scene(width, height, fx, baseline=0.22):
    rig = sn.StereoRig(fx=fx, fy=fx, u0=(width - 1) / 2, v0=(height - 1) / 2,
                       baseline=baseline)
    prims = [sn.Plane([0, -1, 0], -1.6), sn.Box([-8, -2, 12], [-3, 1.6, 30]),
             sn.Box([2.5, -1, 8], [4.5, 1.6, 12]), sn.Box([-1.5, -0.5, 40], [1.5, 1.6, 44]),
             sn.Plane([0, 0, -1], -120)]
    return rig, sn.raycast(sn.SceneSpec(rig=rig, width=width, height=height, primitives=prims))


SQUARE = lambda k: sn.KernelSpec.square(k)  # noqa: E731
CROSS4 = np.array([[1, 0], [-1, 0], [0, 1], [0, -1]])
SPARSE5 = np.array([[0, 0], [2, 1], [1, 2], [-2, -1], [3, -2]])
ASYM6 = np.array([[0, 0], [1, 0], [2, 0], [0, 1], [0, 2], [1, 1]])
SPARSE6 = np.array([[0, 0], [2, 1], [1, 2], [-2, -1], [3, -2], [-1, 3]])


def fixed_cases():
    rig_k = sn.StereoRig(fx=800.0, fy=800.0, u0=31.5, v0=23.5, baseline=0.4)
    rng = np.random.default_rng(1234)
    cases = []
    cases.append(("const", np.full((12, 14), 7.5), SQUARE(3), rig_k))
    cases.append(("hramp", ramp(10, 16, 5.0, 0.2, 0.0), SQUARE(3), rig_k))
    cases.append(("vramp", ramp(10, 16, 5.0, 0.0, 0.3), SQUARE(3), rig_k))
    cases.append(("border5", ramp(12, 12, 1.0, 0.1, 0.1), SQUARE(5), rig_k))
    vals = np.random.default_rng(4).uniform(10, 20, (20, 24))
    vals[7, 9] = np.nan
    cases.append(("hole", vals, SQUARE(3), rig_k))
    cases.append(("asym", ramp(10, 12, 2.0, 0.5, -0.25), sn.KernelSpec(ASYM6), rig_k))
    cases.append(("tiny", np.full((4, 4), 5.0), SQUARE(9), rig_k))
    for i, spec in enumerate([SQUARE(3), SQUARE(5), SQUARE(9), sn.KernelSpec(CROSS4),
                              sn.KernelSpec(SPARSE5), sn.KernelSpec(SPARSE6), SQUARE(15)]):
        v = rng.uniform(1, 50, (40, 44))
        v[rng.random(v.shape) < 0.04] = np.nan
        cases.append((f"rand{i}", v, spec, rig_k))
    # non-positive / non-finite quirks: a finite non-positive
    # neighbour is a valid sample; only the centre needs d > 0
    v = rng.uniform(5, 30, (24, 28))
    v[5, 6] = -2.0
    v[10, 10] = 0.0
    v[15, 3] = np.inf
    v[18, 20] = -np.inf
    v[3, 22] = np.nan
    v[12, 14] = -7.5
    cases.append(("quirks", v, SQUARE(3), rig_k))
    cases.append(("quirks9", v, SQUARE(9), rig_k))
    # exactness fixture: tilted plane (test_kernels.py:184-192)
    n = np.array([0.25, -0.4, -1.0])
    gt = sn.make_plane_scene(n / np.linalg.norm(n), -5.0, rig_k, width=64, height=48)
    cases.append(("plane", gt.disparity.values, SQUARE(5), rig_k))
    # realistic crops: street scene (C3/C4 recipe at reduced size)
    rig_s, gts = street_scene(256, 128, fx=256.0)
    noisy = sn.add_gaussian_noise(gts.disparity, 0.2, seed=3).values
    for k in (3, 9, 15):
        cases.append((f"street_k{k}", noisy, SQUARE(k), rig_s))
    noisy1 = sn.add_gaussian_noise(gts.disparity, 1.0, seed=5).values.copy()
    holes = ndimage.binary_dilation(np.random.default_rng(1005).random(noisy1.shape) < 0.002,
                                    iterations=3)
    noisy1[holes] = np.nan
    cases.append(("street_holes_k9", noisy1, SQUARE(9), rig_s))
    # sphere crop with background (rays that miss are NaN)
    rig_p = sn.StereoRig(fx=128.0, fy=128.0, u0=63.5, v0=63.5, baseline=0.3)
    gtp = sn.raycast(sn.SceneSpec(rig=rig_p, width=128, height=128,
                                  primitives=[sn.Sphere([0, 0, 3], 1.4)]))
    cases.append(("sphere_k9", sn.add_gaussian_noise(gtp.disparity, 0.2, seed=7).values,
                  SQUARE(9), rig_p))
    # odd sizes (no TMA-friendly strides)
    cases.append(("odd_k5", rng.uniform(2, 9, (37, 53)), SQUARE(5), rig_k))
    # genuinely float64 input (not fp32-representable)
    cases.append(("rand_f64", rng.uniform(1, 50, (33, 35)), SQUARE(7), rig_k))
    return cases


def write_fixed():
    store = {}
    names = []
    for name, vals, spec, rig in fixed_cases():
        d = np.asarray(vals, dtype=np.float64)
        if not name.endswith("_f64"):
            d = f32(d)
        field = sn.ScalarField.from_array(d)
        kern = sn.build_kernels(spec)
        aff = sn.convolve_affine(field, kern)
        nf = sn.estimate_normals_fixed(field, rig, kern)
        pts = sn.triangulate_grid(field, rig)
        p = f"{name}__"
        store[p + "d"] = d
        store[p + "offsets"] = np.asarray(spec.offsets, dtype=np.int32)
        store[p + "rig"] = np.array([rig.fx, rig.fy, rig.u0, rig.v0, rig.baseline])
        store[p + "a1"] = aff.a1
        store[p + "a2"] = aff.a2
        store[p + "amask"] = aff.mask
        store[p + "normals"] = nf.vectors
        store[p + "nmask"] = nf.mask
        store[p + "points"] = pts
        names.append(name)
    store["names"] = np.array(names)
    np.savez_compressed(OUT / "fixed_cases.npz", **store)
    return names


def min_index_labels(p):
    """Independent relabel: scipy label, then per-component minimum found by
    an explicit scan (not the oracle's vectorised path)."""
    lab, n = ndimage.label(p, structure=np.ones((3, 3), dtype=bool))
    out = np.full(p.shape, -1, dtype=np.int64)
    flat = lab.ravel()
    seen = {}
    for i in np.flatnonzero(flat):
        c = flat[i]
        if c not in seen:
            seen[c] = i
    for c, first in seen.items():
        out.ravel()[flat == c] = first
    return out


def write_ccl():
    store = {}
    names = []
    rig_s, gts = street_scene(192, 96, fx=192.0)
    cases = []
    for seed, sigma in ((11, 1.0), (12, 0.2)):
        noisy = sn.add_gaussian_noise(gts.disparity, sigma, seed=seed).values.copy()
        holes = ndimage.binary_dilation(
            np.random.default_rng(1000 + seed).random(noisy.shape) < 0.002, iterations=3)
        noisy[holes] = np.nan
        for t in (0.05, 0.2, 1.0):
            cases.append((f"street_s{seed}_t{t}", noisy, rig_s, t))
    step = np.full((8, 10), 5.0)
    step[:, 5:] = 7.0
    rig_d = sn.StereoRig(fx=1.0, fy=1.0, u0=0.0, v0=0.0, baseline=1.0)  # z = 1/d
    cases.append(("step_depth", 1.0 / step, rig_d, 1.9))
    rng = np.random.default_rng(77)
    v = rng.uniform(20, 30, (60, 80))
    v[rng.random(v.shape) < 0.05] = np.nan
    v[30, 40] = -1.0
    cases.append(("random", v, sn.StereoRig(fx=500, fy=500, u0=40, v0=30, baseline=0.3), 0.01))
    for name, vals, rig, t in cases:
        d = f32(vals)
        field = sn.ScalarField.from_array(d)
        depth = sn.depth_field(field, rig)
        edges = sn.depth_laplacian(depth)
        with np.errstate(invalid="ignore"):
            pas = edges.mask & (edges.values <= t)
        p = f"{name}__"
        store[p + "d"] = d
        store[p + "rig"] = np.array([rig.fx, rig.fy, rig.u0, rig.v0, rig.baseline])
        store[p + "t"] = np.array(t)
        store[p + "edges"] = edges.values
        store[p + "emask"] = edges.mask
        store[p + "passable"] = pas
        store[p + "labels"] = min_index_labels(pas)
        names.append(name)
    store["names"] = np.array(names)
    np.savez_compressed(OUT / "ccl_cases.npz", **store)
    return names


def write_accuracy():
    """Reference accuracy on the shipped sphere scene (acceptance criterion 4
    inputs), used as an end-to-end anchor for the device path."""
    scene = sn.load_scene(REF.parent / "scenes" / "sphere.scn")
    gt = sn.raycast(scene)
    rows = []
    for sigma in (0.2, 1.0):
        noisy = sn.add_gaussian_noise(gt.disparity, sigma, seed=7)
        d32 = sn.ScalarField.from_array(f32(noisy.values))
        for k in (9, 15):
            est = sn.estimate_normals_fixed(d32, scene.rig, k)
            st = sn.summarize(sn.angular_error_map(est, gt.normals))
            rows.append({"sigma": sigma, "k": k, "avg_deg": st.avg,
                         "valid_count": st.valid_count, "max_deg": st.max})
    (OUT / "accuracy.json").write_text(json.dumps(
        {"scene": "pkg/scenes/sphere.scn", "seed": 7, "input": "fp32-rounded disparity",
         "rows": rows}, indent=1) + "\n")
    return rows


if __name__ == "__main__":
    print("fixed:", write_fixed())
    print("ccl:", write_ccl())
    print("accuracy:", write_accuracy())
