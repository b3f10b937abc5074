"""CPU checks of the float64 golden fixtures (make_golden_f64.py): the
regenerated inputs are the reference's, the fixtures really separate fp64
from fp32 decisions, the oracle matches them, and the host-side star_trace /
estimate_affine_adaptive (paper_2504_15121_b200/adaptive.py) reproduce the
reference's supports and fits."""

import numpy as np
import pytest

from conftest import f64_input


def _unpack(bits, shape):
    return np.unpackbits(bits, count=shape[0] * shape[1]).reshape(shape).astype(bool)


def test_inputs_regenerate(f64_golden):
    meta, _ = f64_golden
    for e in meta["frames"] + meta["adaptive"]:
        f64_input(e)  # asserts the SHA-256


def test_fixture_separates_fp32_from_fp64(f64_golden):
    """Rounding the inputs to fp32 flips passable pixels on these frames
    (2 pixels at t = 0.2 on the 1024x512 seed-3 frame)."""
    meta, _ = f64_golden
    assert meta["flips"]["street_1024_s02_seed3@0.2"] == 2
    assert sum(meta["flips"].values()) >= 10


def test_oracle_matches_f64_golden(f64_golden):
    from helpers import orig_of
    from oracle import stereonorm_oracle as orc
    meta, arr = f64_golden
    for e in meta["frames"]:
        d, rig = f64_input(e)
        r = orc.Rig(rig.fx, rig.fy, rig.u0, rig.v0, rig.baseline)
        for t in (0.05, 0.2, 1.0):
            p = orc.passable(d, r, t)
            assert np.array_equal(p, _unpack(arr[f"{e['name']}__pass_{t}"], d.shape)), (e["name"], t)
        t = e["ties"][2]
        lab = orc.ccl_labels(d, r, t)
        assert np.array_equal(lab, arr[f"{e['name']}__tie_labels"].astype(np.int64))


def test_star_trace_matches_reference(f64_golden):
    import paper_2504_15121_b200 as sn
    from paper_2504_15121_b200.fields import ScalarField
    from oracle import stereonorm_oracle as orc
    meta, _ = f64_golden
    for a in meta["adaptive"]:
        d, rig = f64_input(a)
        conf = sn.StarConfig(**a["config"])
        field = ScalarField.from_array(d)
        # depth / edge fields from the oracle (pinned to the reference)
        z, zm = orc.depth_field(d, orc.Rig(rig.fx, rig.fy, rig.u0, rig.v0, rig.baseline))
        depth = ScalarField(z, zm)
        edges = None
        if conf.stop == "st":
            e, em = orc.depth_laplacian(z, zm)
            edges = ScalarField(e, em)
        for tr in a["traces"]:
            off = sn.star_trace(tuple(tr["pixel"]), depth, edges, conf)
            assert off.dtype == np.int64
            assert off.tolist() == tr["offsets"], (a["name"], tr["pixel"])
            a1, a2 = sn.estimate_affine_adaptive(field, depth, edges, tuple(tr["pixel"]), conf)
            np.testing.assert_equal(np.array([a1, a2]), np.array([tr["a1"], tr["a2"]]))


def test_star_trace_requires_edges_for_st():
    import paper_2504_15121_b200 as sn
    from paper_2504_15121_b200.fields import ScalarField
    f = ScalarField.from_array(np.ones((4, 4)))
    with pytest.raises(ValueError, match="requires an edge map"):
        sn.star_trace((1, 1), f, None, sn.StarConfig(stop="st"))
