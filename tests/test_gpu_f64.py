"""The float64 paths on the device against the reference's outputs on its own
float64 inputs (tests/golden/make_golden_f64.py): passable sets and edge
values, component labels, adaptive star-fill masks -- all bit-exact -- and
the element-wise geometry (disparity_to_depth, triangulate,
triangulate_grid, depth_field, depth_laplacian) bit-exact in fp64.  Through
the C ABI (device.*) and the drop-in host API (ScalarField in, numpy out)."""

import numpy as np
import pytest
import torch

from conftest import f64_input
from helpers import max_angle_deg, rig_of

pytestmark = pytest.mark.gpu

FRAMES = ["street_1024_s02_seed3", "street_512_s10_holes_seed5", "street_512_s02_seed11"]


def _entry(meta, name, kind="frames"):
    return next(e for e in meta[kind] if e["name"] == name)


def _unpack(bits, shape):
    return np.unpackbits(bits, count=shape[0] * shape[1]).reshape(shape).astype(bool)


def _bits_to_bool(bits, W):
    b = bits.cpu().numpy().view(np.uint32)
    B, H, WW = b.shape
    out = ((b[..., None] >> np.arange(32, dtype=np.uint32)) & 1).astype(bool)
    return out.reshape(B, H, WW * 32)[..., :W]


def _same(a, b):
    """bit-identical float arrays (NaN == NaN, -0.0 != 0.0)"""
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64) if a.size else a,
                                                 b.view(np.uint64) if b.size else b)


def _same_nan(a, b):
    """equal values, NaN positions equal (any NaN payload)"""
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(a, b, equal_nan=True)


@pytest.mark.parametrize("name", FRAMES)
def test_passable_and_labels_f64(f64_golden, cuda_dev, name):
    from paper_2504_15121_b200 import device
    meta, arr = f64_golden
    e = _entry(meta, name)
    d, rig = f64_input(e)
    dt = torch.from_numpy(d).to(cuda_dev)
    for key, t in [(f"pass_{t}", t) for t in (0.05, 0.2, 1.0)] + \
                  [(f"tie_{i}", t) for i, t in enumerate(e["ties"])]:
        want = _unpack(arr[f"{name}__{key}"], d.shape)
        got = _bits_to_bool(device.passable_bits(dt, rig, t), d.shape[1])[0]
        assert np.array_equal(got, want), (key, np.argwhere(got != want)[:5])
        p8 = device.passable(dt, rig, t)[0].cpu().numpy().astype(bool)
        assert np.array_equal(p8, want), key
    for t in (0.05, 0.2, 1.0):
        lab = device.component_labels(dt, rig, t)[0].cpu().numpy()
        assert np.array_equal(lab, arr[f"{name}__labels_{t}"]), t
    lab = device.component_labels(dt, rig, e["ties"][2])[0].cpu().numpy()
    assert np.array_equal(lab, arr[f"{name}__tie_labels"])


@pytest.mark.parametrize("name", FRAMES)
def test_drop_in_components_f64(f64_golden, cuda_dev, name):
    """label_components / passable_set / edge_map on a ScalarField built from
    the reference's float64 values: no fp32 cast anywhere."""
    import paper_2504_15121_b200 as sn
    from paper_2504_15121_b200 import ScalarField
    meta, arr = f64_golden
    e = _entry(meta, name)
    d, rig = f64_input(e)
    f = ScalarField.from_array(d)
    assert np.array_equal(sn.label_components(f, rig, 0.2), arr[f"{name}__labels_0.2"])
    assert np.array_equal(sn.passable_set(f, rig, e["ties"][1]),
                          _unpack(arr[f"{name}__tie_1"], d.shape))
    if f"{name}__edges" in arr:
        em = sn.edge_map(f, rig)
        assert _same_nan(em.values, arr[f"{name}__edges"])
        assert np.array_equal(em.mask, ~np.isnan(arr[f"{name}__edges"]))


@pytest.mark.parametrize("name", FRAMES[1:])
def test_pipeline_f64(f64_golden, cuda_dev, name):
    """sn_pipeline_ws_f64 (fused pass + bits + labels) and the host-buffer
    entry sn_pipeline_host_f64 (pageable numpy input) give the reference's
    labels and the fp64 fused pass's records."""
    import paper_2504_15121_b200 as sn
    from paper_2504_15121_b200 import device
    meta, arr = f64_golden
    e = _entry(meta, name)
    d, rig = f64_input(e)
    dt = torch.from_numpy(np.stack([d, d[::-1].copy()])).to(cuda_dev)
    pts, lab = device.pipeline(dt, rig, 9, 0.2)
    assert np.array_equal(lab[0].cpu().numpy(), arr[f"{name}__labels_0.2"])
    ref = device.oriented_points(dt, rig, 9)
    assert torch.equal(torch.nan_to_num(pts, 7.0), torch.nan_to_num(ref, 7.0))
    hp, hl = sn.oriented_point_cloud(dt.cpu().numpy(), rig, 9, 0.2)
    assert np.array_equal(hl, lab.cpu().numpy())
    assert np.array_equal(np.nan_to_num(hp, nan=7.0), np.nan_to_num(pts.cpu().numpy(), nan=7.0))


ADAPTIVE = ["st_t1_s005", "st_t02_s02", "st_holes", "cd_t01", "cd_shared", "cd_holes_d16"]


@pytest.mark.parametrize("name", ADAPTIVE)
def test_adaptive_f64(f64_golden, cuda_dev, name):
    import paper_2504_15121_b200 as sn
    from paper_2504_15121_b200 import ScalarField, StarConfig
    meta, arr = f64_golden
    a = _entry(meta, name, "adaptive")
    d, rig = f64_input(a)
    nf = sn.estimate_normals_adaptive(ScalarField.from_array(d), rig, StarConfig(**a["config"]))
    want = arr[f"{name}__nmask"]
    assert np.array_equal(nf.mask, want), np.argwhere(nf.mask != want)[:5]
    assert max_angle_deg(nf.vectors[want], arr[f"{name}__normals"][want]) < 1e-4


def test_geometry_f64(f64_golden, cuda_dev):
    import paper_2504_15121_b200 as sn
    meta, arr = f64_golden
    rig = rig_of(arr["geom__rig"])
    d = arr["geom__d"]
    assert _same_nan(sn.disparity_to_depth(d, rig), arr["geom__depth"])
    x, y, z = sn.triangulate(arr["geom__u"], arr["geom__v"], d, rig)
    assert _same_nan(x, arr["geom__x"]) and _same_nan(y, arr["geom__y"])
    assert _same_nan(z, arr["geom__z"])
    xb, yb, zb = sn.triangulate(arr["geom__u"][:7], 42.0, d[:11, None], rig)
    assert xb.shape == arr["geom__bx"].shape and yb.shape == arr["geom__by"].shape
    assert zb.shape == arr["geom__bz"].shape
    assert _same_nan(xb, arr["geom__bx"]) and _same_nan(yb, arr["geom__by"])
    assert _same_nan(zb, arr["geom__bz"])
    z0 = sn.disparity_to_depth(77.25, rig)
    assert np.isscalar(z0) or np.ndim(z0) == 0
    assert z0 == arr["geom__depth"][13]


def test_grid_geometry_f64(f64_golden, cuda_dev):
    import paper_2504_15121_b200 as sn
    from paper_2504_15121_b200 import ScalarField
    _, arr = f64_golden
    rig = rig_of(arr["grid__rig"])
    f = ScalarField.from_array(arr["grid__d"])
    pts = sn.triangulate_grid(f, rig)
    assert pts.dtype == np.float64 and _same_nan(pts, arr["grid__points"])
    df = sn.depth_field(f, rig)
    assert _same_nan(df.values, arr["grid__depth"]) and np.array_equal(df.mask, arr["grid__depth_mask"])
    lap = sn.depth_laplacian(df)
    assert _same_nan(lap.values, arr["grid__lap"]) and np.array_equal(lap.mask, arr["grid__lap_mask"])


def test_fp32_inputs_unchanged(cuda_dev):
    """fp32 tensors stay on the fp32 fast path and agree with the fp64 path on
    the same (fp32-representable) values."""
    from paper_2504_15121_b200 import device, scenes
    sc = scenes.street_scene(256, 128)
    d = scenes.add_gaussian_noise(scenes.raycast(sc)[0], 0.5, 3).astype(np.float32)
    d32 = torch.from_numpy(d).to(cuda_dev)
    d64 = d32.double()
    for t in (0.05, 0.2, 1.0):
        assert torch.equal(device.passable_bits(d32, sc.rig, t), device.passable_bits(d64, sc.rig, t))
        assert torch.equal(device.component_labels(d32, sc.rig, t),
                           device.component_labels(d64, sc.rig, t))


@pytest.mark.parametrize("pick", ["ties", "out_of_fp32_range", "tiny_shapes"])
def test_f64_filter_edge_cases(cuda_dev, pick):
    """fp64 inputs the fp32 filter cannot decide: thresholds equal to edge
    values of float64 disparities that fp32 cannot represent, samples outside
    fp32's range (1e-300, 1e300, fp64 subnormals, -0.0, +-inf), and frames
    too small to hold an interior pixel -- bits, labels, pipeline and the
    star-fill masks all equal the oracle's fp64 decisions."""
    from oracle import stereonorm_oracle as orc
    from paper_2504_15121_b200 import StarConfig, device, scenes
    shapes = [(96, 200)] if pick != "tiny_shapes" else [(1, 1), (2, 2), (3, 3), (3, 40), (40, 3),
                                                        (4, 5)]
    for H, W in shapes:
        sc = scenes.street_scene(max(W, 8), max(H, 8))
        d = scenes.add_gaussian_noise(scenes.raycast(sc)[0], 0.7, 11)[:H, :W].copy()
        rng = np.random.default_rng(H * 1000 + W)
        if pick == "out_of_fp32_range":
            sel = rng.random(d.shape)
            d[sel < 0.02] = 1e-300
            d[(sel >= 0.02) & (sel < 0.04)] = 1e300
            d[(sel >= 0.04) & (sel < 0.05)] = 5e-324
            d[(sel >= 0.05) & (sel < 0.06)] = -0.0
            d[(sel >= 0.06) & (sel < 0.07)] = np.inf
            d[(sel >= 0.07) & (sel < 0.08)] = -np.inf
            d[(sel >= 0.08) & (sel < 0.09)] = np.nan
            d[(sel >= 0.09) & (sel < 0.10)] = 3.0e-39  # fp32 subnormal range
        o = orc.Rig(sc.rig.fx, sc.rig.fy, sc.rig.u0, sc.rig.v0, sc.rig.baseline)
        e, em = orc.depth_laplacian(*orc.depth_field(d, o))
        ts = [0.05, 0.2, 1.0]
        if pick == "ties" and em.any():
            vals = np.sort(e[em])
            ts += [float(vals[len(vals) // 5]), float(vals[len(vals) // 2]), float(vals[-1])]
        dt = torch.from_numpy(d).to(cuda_dev)
        for t in ts:
            want = orc.passable(d, o, t)
            got = _bits_to_bool(device.passable_bits(dt, sc.rig, t), W)[0]
            assert np.array_equal(got, want), (H, W, t)
            lab = device.component_labels(dt, sc.rig, t)[0].cpu().numpy().astype(np.int64)
            assert np.array_equal(lab, orc.ccl_labels(d, o, t)), (H, W, t)
            if H * W >= 9:
                _, lab2 = device.pipeline(dt, sc.rig, 3, t)
                assert np.array_equal(lab2[0].cpu().numpy().astype(np.int64), lab), (H, W, t)
        for cfg in (orc.Star(stop="st", threshold=0.5), orc.Star(stop="cd", threshold=0.1)):
            n_ref, ok_ref = orc.estimate_normals_adaptive(d, o, cfg)
            mask = torch.empty((1, H, W), dtype=torch.uint8, device=cuda_dev)
            device.adaptive_points(dt, sc.rig, StarConfig(stop=cfg.stop, threshold=cfg.threshold),
                                   mask=mask)
            assert np.array_equal(mask[0].cpu().numpy().astype(bool), ok_ref), (H, W, cfg)


@pytest.mark.parametrize("shape", [(0, 16, 32), (2, 0, 32), (2, 16, 0)])
def test_empty_inputs_f64(cuda_dev, shape):
    from paper_2504_15121_b200 import StarConfig, StereoRig, device
    rig = StereoRig(100.0, 100.0, 8.0, 8.0, 0.2)
    d = torch.empty(shape, dtype=torch.float64, device=cuda_dev)
    B, H, W = shape
    assert device.oriented_points(d, rig, 3).shape == (B, H, W, 6)
    assert device.passable_bits(d, rig, 0.2).shape == (B, H, device.bit_words(W))
    assert device.component_labels(d, rig, 0.2).shape == (B, H, W)
    pts, lab = device.pipeline(d, rig, 3, 0.2)
    assert pts.shape == (B, H, W, 6) and lab.shape == (B, H, W)
    assert device.adaptive_points(d, rig, StarConfig(stop="st", threshold=0.1)).shape == (B, H, W, 6)
    p8, e = device.passable(d, rig, 0.2, edges=torch.empty(shape, dtype=torch.float64,
                                                             device=cuda_dev))
    assert p8.shape == (B, H, W) and e.shape == (B, H, W)
    torch.cuda.synchronize()
