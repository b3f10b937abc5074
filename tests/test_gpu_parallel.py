"""Partition invariance on the device (reference test_parallel.py:48-75,
restated for strips and frame shards): strip-partitioned points and labels
are bit-identical to the whole-frame result, for any strip count; frame
shards reproduce the whole batch."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _nan_eq(a, b):
    return torch.equal(torch.nan_to_num(a, 7.0), torch.nan_to_num(b, 7.0))


@pytest.mark.parametrize("n_strips,k", [(2, 9), (3, 9), (8, 9), (5, 15), (4, 3)])
def test_strip_frame_matches_whole_frame(cuda_dev, n_strips, k):
    from scipy import ndimage
    from paper_2504_15121_b200 import device, scenes
    from paper_2504_15121_b200.parallel import StripPlan, local_strip_frame
    sc = scenes.street_scene(768, 432)
    d = scenes.add_gaussian_noise(scenes.raycast(sc)[0], 1.0, 5)
    holes = ndimage.binary_dilation(np.random.default_rng(3).random(d.shape) < 0.002, iterations=2)
    d[holes] = np.nan
    dt = torch.from_numpy(d.astype(np.float32)).to(cuda_dev)
    plan = StripPlan.for_kernel(432, 768, n_strips, k)
    for t in (0.05, 1.0):
        pts, lab = local_strip_frame(dt, plan, sc.rig, k, t)
        whole_pts = device.oriented_points(dt, sc.rig, k)[0]
        whole_lab = device.component_labels(dt, sc.rig, t)[0]
        assert _nan_eq(pts, whole_pts)
        assert torch.equal(lab, whole_lab)


def test_frame_shards_match_batch(cuda_dev):
    from paper_2504_15121_b200 import device, scenes
    from paper_2504_15121_b200.parallel import shard_range
    sc = scenes.street_scene(512, 256)
    clean = scenes.raycast(sc)[0]
    frames = np.stack([scenes.add_gaussian_noise(clean, 0.2, i) for i in range(7)])
    d = torch.from_numpy(frames.astype(np.float32)).to(cuda_dev)
    whole = device.oriented_points(d, sc.rig, 9)
    whole_lab = device.component_labels(d, sc.rig, 0.2)
    for world in (2, 3, 4):
        for r in range(world):
            a, b = shard_range(7, r, world)
            if a == b:
                continue
            assert _nan_eq(device.oriented_points(d[a:b], sc.rig, 9), whole[a:b])
            assert torch.equal(device.component_labels(d[a:b], sc.rig, 0.2), whole_lab[a:b])


def test_host_pipeline_matches_device(cuda_dev):
    """sn_pipeline_host (chunked H2D / compute / D2H) == the device pipeline,
    with a batch that spans several chunks and an odd last chunk."""
    import paper_2504_15121_b200 as sn
    from paper_2504_15121_b200 import device, scenes
    sc = scenes.street_scene(2048, 1024)
    clean = scenes.raycast(sc)[0]
    frames = np.stack([scenes.add_gaussian_noise(clean, 0.3, i) for i in range(11)]).astype(np.float32)
    frames[3, 100:140, 500:560] = np.nan
    pts, lab = sn.oriented_point_cloud(frames, sc.rig, 9, 0.2)
    dp, dl = device.pipeline(torch.from_numpy(frames).to(cuda_dev), sc.rig, 9, 0.2)
    assert np.array_equal(np.nan_to_num(pts, nan=7.0), np.nan_to_num(dp.cpu().numpy(), nan=7.0))
    assert np.array_equal(lab, dl.cpu().numpy())


def test_c5_eight_strips(cuda_dev):
    """C5: one 7680x4320 street frame split into 8 strips of
    540 rows -- points and labels bit-identical to the whole frame, labels
    equal to the oracle's, normals of an interior crop within 1e-4 deg of the
    oracle's."""
    from helpers import max_angle_deg
    from oracle import stereonorm_oracle as orc
    from paper_2504_15121_b200 import device, scenes
    from paper_2504_15121_b200.parallel import StripPlan, local_strip_frame
    sc = scenes.street_scene(7680, 4320)
    d = scenes.add_gaussian_noise(scenes.raycast(sc)[0], 0.2, 0).astype(np.float32)
    dt = torch.from_numpy(d).to(cuda_dev)
    plan = StripPlan.for_kernel(4320, 7680, 8, 9)
    assert [plan.owned(g) for g in range(8)] == [(540 * g, 540 * (g + 1)) for g in range(8)]
    pts, lab = local_strip_frame(dt, plan, sc.rig, 9, 0.2)
    whole = device.oriented_points(dt, sc.rig, 9)[0]
    whole_lab = device.component_labels(dt, sc.rig, 0.2)[0]
    assert _nan_eq(pts, whole)
    assert torch.equal(lab, whole_lab)
    r = sc.rig
    orig = orc.Rig(r.fx, r.fy, r.u0, r.v0, r.baseline)
    assert np.array_equal(whole_lab.cpu().numpy().astype(np.int64),
                          orc.ccl_labels(d.astype(np.float64), orig, 0.2))
    # normals: a crop across the strip seam at row 2160 (4-row halo for k = 9)
    crop = d[2100:2220].astype(np.float64)
    ref6, ok = orc.oriented_points(crop, orc.Rig(r.fx, r.fy, r.u0, r.v0 - 2100, r.baseline), 9)
    got = whole[2104:2216].cpu().numpy()
    okc = ok[4:-4]
    assert np.array_equal(np.isfinite(got[..., 3:]).all(-1), okc)
    assert max_angle_deg(got[okc][:, 3:], ref6[4:-4][okc][:, 3:]) < 1e-4


def test_device_seam_merge_matches_host(cuda_dev):
    """sn_seam_merge (device, the multi-GPU strip path's merge) gives the
    same roots as sn_seam_merge_host for every seam label, on random seam
    rows with 8-connected contacts, including labels that chain across
    several strips."""
    from paper_2504_15121_b200 import device
    rng = np.random.default_rng(3)
    for n_strips, W in ((2, 64), (5, 300), (8, 7680)):
        H = n_strips * 10
        seams = np.full((n_strips, 2, W), -1, np.int32)
        for s in range(n_strips):
            for r in range(2):
                row = s * 10 + (0 if r == 0 else 9)
                on = rng.random(W) < 0.6
                # labels: some raster index of a pixel at or before this row
                seams[s, r][on] = rng.integers(0, row * W + 1, on.sum())
        keys, vals = device.seam_merge(seams)
        table = device.seam_table(torch.from_numpy(seams).to(cuda_dev), H * W).cpu().numpy()
        want = {int(k): int(v) for k, v in zip(keys, vals)}
        for v in np.unique(seams[seams >= 0]):
            assert table[v] == want.get(int(v), int(v)), (n_strips, W, v)
        lab = torch.from_numpy(seams.reshape(-1).copy()).to(cuda_dev)
        device.relabel_table(lab, torch.from_numpy(table).to(cuda_dev))
        got = lab.cpu().numpy()
        ref = np.array([want.get(int(v), int(v)) if v >= 0 else -1 for v in seams.reshape(-1)])
        assert np.array_equal(got, ref)
