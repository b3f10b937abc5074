"""CPU-only checks: C-ABI library loads and exports every declared symbol,
host-side validation mirrors the reference, scene synthesis reproduces the
reference inputs, seam merge logic (host C++) vs the oracle labeller."""

import re
from pathlib import Path

import numpy as np
import pytest

import paper_2504_15121_b200 as sn
from paper_2504_15121_b200 import _native, scenes

ROOT = Path(__file__).resolve().parent.parent


def test_library_exports_every_header_symbol():
    lib = _native.load()
    header = (ROOT / "include" / "sn_b200.h").read_text()
    names = re.findall(r"SN_API\s+(?:int|const char\*)\s+(sn_\w+)\(", header)
    assert len(names) >= 16
    for n in names:
        assert hasattr(lib, n), n
        assert n in _native.SIGNATURES, f"{n} has no ctypes signature"
    assert lib.sn_abi_version() == 2


def test_kernel_moments_match_build_kernels():
    for k in (3, 5, 9, 15):
        m = _native.kernel_moments(sn.KernelSpec.square(k).offsets)
        kk = sn.build_kernels(sn.KernelSpec.square(k))
        assert (m.alpha, m.beta, m.gamma, m.det) == (kk.alpha, kk.beta, kk.gamma, kk.det)
        assert m.square_r == k // 2
    m = _native.kernel_moments([[0, 0], [1, 0], [2, 0], [0, 1], [0, 2], [1, 1]])
    assert m.square_r == -1 and m.sx == 4 and m.sy == 4
    with pytest.raises(sn.DegenerateSupportError):
        _native.kernel_moments([[-1, 0], [0, 0], [1, 0]])
    with pytest.raises(ValueError):
        _native.kernel_moments([[0, 0], [0, 0]])


def test_build_kernels_kats():
    k = sn.build_kernels(sn.KernelSpec.square(3))
    assert (k.alpha, k.beta, k.gamma) == (6.0, 0.0, 6.0)
    assert np.array_equal(k.s1, k.spec.offsets[:, 0] / 6.0)
    assert k.delta1 == 0.0 and k.delta2 == 0.0
    assert sn.build_kernels(sn.KernelSpec.square(5)).alpha == 50.0
    with pytest.raises(sn.DegenerateSupportError):
        sn.build_kernels(sn.KernelSpec(np.array([[-1, 0], [0, 0], [1, 0]])))
    rng = np.random.default_rng(9)
    for _ in range(20):
        off = np.unique(rng.integers(-4, 5, size=(rng.integers(3, 12), 2)), axis=0)
        try:
            k = sn.build_kernels(sn.KernelSpec(off))
        except sn.DegenerateSupportError:
            continue
        v = off.astype(float)
        s = np.linalg.solve(v.T @ v, v.T)
        assert np.allclose(k.s1, s[0], rtol=1e-12, atol=1e-14)
        assert np.allclose(k.s2, s[1], rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("width", [1, 2, 4, -3])
def test_square_rejects_bad_width(width):
    with pytest.raises(ValueError):
        sn.KernelSpec.square(width)


def test_rig_and_estimator_protocol():
    with pytest.raises(ValueError):
        sn.StereoRig(fx=-1, fy=1, u0=0, v0=0, baseline=1)
    with pytest.raises(ValueError):
        sn.StereoRig(fx=1, fy=1, u0=0, v0=0, baseline=0)
    rig = sn.StereoRig(600.0, 600.0, 23.5, 17.5, 0.4)
    est = sn.AffineNormalEstimator(rig, kernel_size=5)
    params = est.get_params()
    assert params == {"rig": rig, "kernel_size": 5, "threads": 1}
    assert type(est)(**params).get_params() == params
    assert est.set_params(kernel_size=9) is est and est.kernel_size == 9
    with pytest.raises(ValueError):
        est.set_params(bogus=1)
    assert est.fit() is est
    assert sn.as_rig({"fx": 10, "fy": 10, "u0": 1, "v0": 2, "baseline": 0.5}).fx == 10
    with pytest.raises(ValueError):
        sn.as_rig([1, 2, 3])
    with pytest.raises(ValueError):
        sn.as_scalar_field(np.zeros(5))


def test_sklearn_clone():
    sklearn = pytest.importorskip("sklearn")
    from sklearn.base import clone
    est = sn.AffineNormalEstimator(sn.StereoRig(600.0, 600.0, 23.5, 17.5, 0.4), kernel_size=5)
    assert clone(est).get_params() == est.get_params()


def test_format_kernel_dump_layout():
    dump = sn.format_kernel_dump(sn.build_kernels(sn.KernelSpec.square(3)))
    assert "alpha 6" in dump and dump.count("vy=") == 6
    dump = sn.format_kernel_dump(sn.build_kernels(sn.KernelSpec(np.array([[1, 0], [0, 1], [-1, -1]]))))
    assert "v=(+1,+0)" in dump


def test_scene_synthesis_reproduces_reference_inputs(fixed_golden):
    sc = scenes.street_scene(256, 128, fx=256.0)
    disp, _, _ = scenes.raycast(sc)
    noisy = scenes.add_gaussian_noise(disp, 0.2, 3).astype(np.float32).astype(np.float64)
    np.testing.assert_array_equal(noisy, fixed_golden["street_k9"]["d"])
    sp = scenes.sphere_scene(128, 128, fx=128.0)
    d2 = scenes.add_gaussian_noise(scenes.raycast(sp)[0], 0.2, 7).astype(np.float32)
    np.testing.assert_array_equal(d2.astype(np.float64), fixed_golden["sphere_k9"]["d"])


def test_seam_merge_matches_full_frame_labels():
    """Strip labelling + host seam merge == labelling the whole frame
    (oracle labeller per strip; the merge is the shipped C++ routine)."""
    from oracle.stereonorm_oracle import label_components
    from paper_2504_15121_b200 import device
    rng = np.random.default_rng(5)
    H, W, n = 96, 70, 4
    p = rng.random((H, W)) < 0.55
    full = label_components(p)
    rows = H // n
    strips = [label_components(p[s * rows:(s + 1) * rows], index_offset=s * rows * W)
              for s in range(n)]
    seams = np.stack([np.stack([s[0], s[-1]]) for s in strips]).astype(np.int32)
    keys, vals = device.seam_merge(seams)
    lut = dict(zip(keys.tolist(), vals.tolist()))
    merged = np.concatenate([np.vectorize(lambda v: lut.get(v, v))(s) for s in strips])
    assert np.array_equal(merged, full)


def test_ply_writer_matches_reference_bytes():
    """formats.ply_from_vertices / write_ply_oriented == the reference writer
    (golden bytes from formats.py:170-185), binary and ASCII, empty clouds."""
    from paper_2504_15121_b200 import formats
    z = np.load(Path(__file__).resolve().parent / "golden" / "ply_cases.npz")
    pts, nrm = z["points"], z["normals"]
    for binary, tag in ((True, "bin"), (False, "ascii")):
        assert formats.write_ply_oriented(pts, nrm, binary) == z[f"ply_{tag}"].tobytes()
        assert formats.ply_from_vertices(np.hstack([pts, nrm]), binary) == z[f"ply_{tag}"].tobytes()
        assert formats.write_ply_oriented(np.zeros((0, 3)), np.zeros((0, 3)), binary) == \
            z[f"empty_{tag}"].tobytes()


def test_c_demo_builds_against_the_abi(tmp_path):
    """examples/sn_demo.c is a plain-C client of include/sn_b200.h: it must
    compile and link against the in-tree library (run on the GPU in
    tests/test_gpu_parity.py::test_c_demo_runs)."""
    import shutil
    import subprocess
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    lib = root / "paper_2504_15121_b200" / "libsn_b200.so"
    if not lib.exists() or shutil.which("gcc") is None:
        pytest.skip("library or gcc missing")
    exe = tmp_path / "sn_demo"
    subprocess.run(["gcc", "-O2", "-Wall", "-Werror", f"-I{root / 'include'}",
                    str(root / "examples" / "sn_demo.c"), f"-L{lib.parent}", "-lsn_b200",
                    f"-Wl,-rpath,{lib.parent}", "-lm", "-o", str(exe)], check=True)
    assert exe.exists()


def _host_golden():
    import json
    from conftest import GOLDEN
    return json.loads((GOLDEN / "host_cases.json").read_text())


def test_format_kernel_dump_matches_reference():
    """format_kernel_dump text identical to the reference's (kernels.py:264-296)."""
    from paper_2504_15121_b200 import KernelSpec, build_kernels, format_kernel_dump
    g = _host_golden()
    specs = {"sq3": KernelSpec.square(3), "sq5": KernelSpec.square(5), "sq9": KernelSpec.square(9),
             "cross4": KernelSpec(np.array([[1, 0], [-1, 0], [0, 1], [0, -1]])),
             "sparse5": KernelSpec(np.array([[0, 0], [2, 1], [1, 2], [-2, -1], [3, -2]])),
             "asym6": KernelSpec(np.array([[0, 0], [1, 0], [2, 0], [0, 1], [0, 2], [1, 1]]))}
    for name, spec in specs.items():
        assert format_kernel_dump(build_kernels(spec)) == g["dumps"][name], name


def test_estimate_affine_direct_matches_reference():
    """Single-pixel solves bit-identical to the reference (kernels.py:206-234)."""
    from paper_2504_15121_b200 import KernelSpec, ScalarField, estimate_affine_direct
    g = _host_golden()
    d = np.array([[np.nan if x is None else x for x in row] for row in g["disparity"]])
    d[0, 0] = np.inf
    field = ScalarField.from_array(d)
    specs = {"sq3": KernelSpec.square(3), "sq5": KernelSpec.square(5), "sq9": KernelSpec.square(9),
             "cross4": KernelSpec(np.array([[1, 0], [-1, 0], [0, 1], [0, -1]])),
             "sparse5": KernelSpec(np.array([[0, 0], [2, 1], [1, 2], [-2, -1], [3, -2]])),
             "asym6": KernelSpec(np.array([[0, 0], [1, 0], [2, 0], [0, 1], [0, 2], [1, 1]]))}
    for c in g["direct"]:
        got = estimate_affine_direct(field, tuple(c["pixel"]), specs[c["spec"]])
        want = tuple(float("nan") if x is None else x for x in (c["a1"], c["a2"]))
        np.testing.assert_equal(np.array(got), np.array(want))


def test_pfm_writers_match_reference_bytes():
    import base64
    from paper_2504_15121_b200 import NormalField, ScalarField, formats
    g = _host_golden()
    d = np.array([[np.nan if x is None else x for x in row] for row in g["disparity"]])
    d[0, 0] = np.inf
    assert formats.write_pfm(ScalarField.from_array(d)) == base64.b64decode(g["pfm"])
    nf = NormalField.from_array(np.array(g["normals"]))
    assert formats.write_pfm_normals(nf) == base64.b64decode(g["pfm_normals"])
