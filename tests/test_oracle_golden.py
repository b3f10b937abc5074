"""Pin the CPU oracle to the reference's own outputs (CPU only).

Golden vectors come from running the reference package (tests/golden/
make_golden.py); the oracle must reproduce them: masks/labels bit-exact,
values to fp64 rounding.
"""

from pathlib import Path

import numpy as np
import pytest

from oracle import stereonorm_oracle as orc
from helpers import orig_of


def test_square_offsets_match_reference_order(fixed_golden):
    for name in ("const", "street_k9", "street_k15"):
        off = fixed_golden[name]["offsets"]
        k = int(round(np.sqrt(len(off))))
        assert np.array_equal(orc.square_offsets(k), off)


@pytest.mark.parametrize("name", ["const", "hramp", "vramp", "border5", "hole", "asym", "tiny",
                                  "rand0", "rand1", "rand2", "rand3", "rand4", "rand5", "rand6",
                                  "quirks", "quirks9", "plane", "street_k3", "street_k9",
                                  "street_k15", "street_holes_k9", "sphere_k9", "odd_k5",
                                  "rand_f64"])
def test_oracle_fixed_matches_reference(fixed_golden, name):
    c = fixed_golden[name]
    rig = orig_of(c["rig"])
    a1, a2, am = orc.convolve_affine(c["d"], c["offsets"])
    assert np.array_equal(am, c["amask"])
    np.testing.assert_allclose(a1[am], c["a1"][am], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(a2[am], c["a2"][am], rtol=1e-12, atol=1e-12)
    n, nm = orc.estimate_normals_fixed(c["d"], rig, c["offsets"])
    assert np.array_equal(nm, c["nmask"])
    np.testing.assert_allclose(n[nm], c["normals"][nm], rtol=1e-10, atol=1e-12)
    assert np.isnan(n[~nm]).all()
    p = orc.triangulate_grid(c["d"], rig)
    assert np.array_equal(np.isfinite(p), np.isfinite(c["points"]))
    fin = np.isfinite(p)
    np.testing.assert_array_equal(p[fin], c["points"][fin])


def test_oracle_thread_invariance(fixed_golden):
    c = fixed_golden["street_holes_k9"]
    rig = orig_of(c["rig"])
    a, am = orc.estimate_normals_fixed(c["d"], rig, 9, threads=1)
    b, bm = orc.estimate_normals_fixed(c["d"], rig, 9, threads=4)
    assert np.array_equal(am, bm)
    assert np.array_equal(a, b, equal_nan=True)


def test_oracle_degenerate_pattern_raises():
    with pytest.raises(ValueError):
        orc.weights(np.array([[-1, 0], [0, 0], [1, 0]]))


@pytest.mark.parametrize("name", ["street_s11_t0.05", "street_s11_t0.2", "street_s11_t1.0",
                                  "street_s12_t0.05", "street_s12_t0.2", "street_s12_t1.0",
                                  "step_depth", "random"])
def test_oracle_ccl_matches_reference(ccl_golden, name):
    c = ccl_golden[name]
    rig = orig_of(c["rig"])
    z, zm = orc.depth_field(c["d"], rig)
    e, em = orc.depth_laplacian(z, zm)
    assert np.array_equal(em, c["emask"])
    np.testing.assert_array_equal(e[em], c["edges"][em])  # bit-exact
    p = orc.passable(c["d"], rig, float(c["t"]))
    assert np.array_equal(p, c["passable"])
    assert np.array_equal(orc.label_components(p), c["labels"])


def test_label_components_kats():
    p = np.zeros((5, 6), bool)
    p[0, 0] = p[1, 1] = p[2, 2] = True          # diagonal chain: one component
    p[4, 5] = True                               # isolated
    p[0, 4] = p[0, 5] = p[1, 5] = True           # L shape
    lab = orc.label_components(p)
    assert lab[2, 2] == 0 and lab[1, 1] == 0
    assert lab[4, 5] == 4 * 6 + 5
    assert lab[1, 5] == 4
    assert (lab[~p] == -1).all()
    assert orc.label_components(p, index_offset=100)[1, 5] == 104


ADAPTIVE = ["street_cd_d8_s10", "street_st_d8_s10", "street_cd_shared", "street_cd_holes",
            "street_st_holes", "sphere_cd_d16_s5", "sphere_st_d3_s2", "sphere_cd_d5_s30",
            "street_cd_s1", "tiny"]


@pytest.mark.parametrize("name", ADAPTIVE)
def test_oracle_adaptive_matches_reference(adaptive_golden, name):
    """The oracle's star-fill restatement == reference estimate_normals_adaptive
    (adaptive.py:177-268), bit for bit (same fp64 op order)."""
    from oracle import stereonorm_oracle as orc
    c = adaptive_golden[name]
    fx, fy, u0, v0, b = (float(v) for v in c["rig"])
    n, ok = orc.estimate_normals_adaptive(c["d"], orc.Rig(fx, fy, u0, v0, b), orc.Star(**c["config"]))
    assert np.array_equal(ok, c["nmask"])
    np.testing.assert_array_equal(n[ok], c["normals"][ok])


def test_oracle_evaluation_matches_reference():
    """The oracle's angular_error_map + summarize == the reference's
    (evaluation.py:34-73) on its own golden cases, bit for bit."""
    from oracle import stereonorm_oracle as orc
    z = np.load(Path(__file__).resolve().parent / "golden" / "eval_cases.npz")
    for tag in z["names"]:
        tag = str(tag)
        err, ok = orc.angular_error_map(z[f"{tag}__est_n"], z[f"{tag}__est_m"], z["gt_n"], z["gt_m"],
                                        z[f"{tag}__mask"])
        ref = z[f"{tag}__err"]
        assert np.array_equal(ok, np.isfinite(ref)), tag
        np.testing.assert_array_equal(err[ok], ref[ok])
        assert orc.summarize(err, ok) == tuple(
            int(v) if i == 5 else float(v) for i, v in enumerate(z[f"{tag}__stats"])), tag
    with pytest.raises(ValueError):
        orc.summarize(np.zeros(3), np.zeros(3, bool))


def test_oracle_codecs_match_reference():
    """The oracle's PNG16 dequantisation and PFM payload decode == the
    reference's read_disparity_png16 / read_pfm (formats.py:84-150) on its own
    golden files, bit for bit."""
    import io
    from PIL import Image
    from oracle import stereonorm_oracle as orc
    from paper_2504_15121_b200.formats import _pfm_header
    z = np.load(Path(__file__).resolve().parent / "golden" / "codec_cases.npz")
    for tag in z["png_names"]:
        tag = "png_" + str(tag)
        raw = np.asarray(Image.open(io.BytesIO(z[f"{tag}__bytes"].tobytes())), dtype=np.int64)
        assert np.array_equal(raw, z[f"{tag}__raw"]), tag
        v, m = orc.dequant_png16(raw, float(z[f"{tag}__scale"]), int(z[f"{tag}__invalid"]))
        assert np.array_equal(m, z[f"{tag}__mask"]), tag
        np.testing.assert_array_equal(v[m], z[f"{tag}__values"][m])
    for tag in z["pfm_names"]:
        tag = "pfm_" + str(tag)
        data = z[f"{tag}__bytes"].tobytes()
        _, w, h, scale, pos = _pfm_header(data)  # the product's host-side header parser
        ch = int(z[f"{tag}__channels"])
        g = orc.decode_pfm_payload(data[pos:pos + w * h * ch * 4], h, w, ch, scale < 0)
        # read_pfm / read_pfm_normals then mask non-finite samples (fields.py:37-46)
        ok = np.isfinite(g) if ch == 1 else np.isfinite(g).all(-1)
        assert np.array_equal(ok, z[f"{tag}__mask"]), tag
        np.testing.assert_array_equal(g[ok], z[f"{tag}__values"][ok])
