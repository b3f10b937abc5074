"""Adaptive star-fill normals on the device vs the reference's golden vectors
(adaptive.py:177-268, tests/golden/make_golden_adaptive.py) and vs the
oracle restatement on larger frames.  Masks bit-exact; normals within the
fp32-storage floor; points identical to the fixed pass's."""

import numpy as np
import pytest
import torch

from helpers import max_angle_deg, rig_of

pytestmark = pytest.mark.gpu

ADAPTIVE = ["street_cd_d8_s10", "street_st_d8_s10", "street_cd_shared", "street_cd_holes",
            "street_st_holes", "sphere_cd_d16_s5", "sphere_st_d3_s2", "sphere_cd_d5_s30",
            "street_cd_s1", "tiny"]


@pytest.mark.parametrize("name", ADAPTIVE)
def test_adaptive_golden(adaptive_golden, cuda_dev, name):
    from paper_2504_15121_b200 import StarConfig, device
    c = adaptive_golden[name]
    rig = rig_of(c["rig"])
    d = torch.from_numpy(c["d"].astype(np.float32)).to(cuda_dev)
    mask = torch.empty((1,) + tuple(d.shape), dtype=torch.uint8, device=cuda_dev)
    out = device.adaptive_points(d, rig, StarConfig(**c["config"]), mask=mask)
    o = out[0].cpu().numpy()
    m = mask[0].cpu().numpy().astype(bool)
    assert np.array_equal(m, c["nmask"]), f"mask differs at {np.argwhere(m != c['nmask'])[:5]}"
    assert np.array_equal(np.isfinite(o[..., 3:]).all(-1), m)
    assert max_angle_deg(o[m][:, 3:], c["normals"][m]) < 1e-4
    fixed = device.oriented_points(d, rig, 3)[0].cpu().numpy()
    assert np.array_equal(np.nan_to_num(o[..., :3], nan=7.0), np.nan_to_num(fixed[..., :3], nan=7.0))


def test_adaptive_reference_api(adaptive_golden, cuda_dev):
    """estimate_normals_adaptive / AdaptiveNormalEstimator on the reference
    signatures return the reference's NaN-row float64 arrays."""
    import paper_2504_15121_b200 as sn
    c = adaptive_golden["street_cd_d8_s10"]
    rig = rig_of(c["rig"])
    nf = sn.estimate_normals_adaptive(sn.ScalarField.from_array(c["d"]), rig,
                                      sn.StarConfig(**c["config"]))
    assert np.array_equal(nf.mask, c["nmask"])
    assert max_angle_deg(nf.vectors[nf.mask], c["normals"][nf.mask]) < 1e-4
    est = sn.AdaptiveNormalEstimator(rig, **c["config"])
    v = est.fit().transform(c["d"])
    assert v.dtype == np.float64 and np.array_equal(np.isfinite(v).all(-1), c["nmask"])


@pytest.mark.parametrize("cfg", [dict(stop="cd", threshold=0.1),
                                 dict(stop="st", threshold=0.2),
                                 dict(stop="cd", threshold=0.2, shared_range=True, directions=12),
                                 dict(stop="st", threshold=1.0, max_steps=30, directions=16)])
def test_adaptive_vs_oracle_street(cuda_dev, cfg):
    """A C4-style frame (noise + dilated holes) at 512x256 against the oracle."""
    from scipy import ndimage
    from oracle import stereonorm_oracle as orc
    from paper_2504_15121_b200 import StarConfig, device, scenes
    sc = scenes.street_scene(512, 256)
    d = scenes.add_gaussian_noise(scenes.raycast(sc)[0], 0.3, 12)
    holes = ndimage.binary_dilation(np.random.default_rng(5).random(d.shape) < 0.002, iterations=2)
    d[holes] = np.nan
    d = d.astype(np.float32)
    r = sc.rig
    n_ref, ok_ref = orc.estimate_normals_adaptive(d.astype(np.float64),
                                                  orc.Rig(r.fx, r.fy, r.u0, r.v0, r.baseline),
                                                  orc.Star(**cfg))
    mask = torch.empty((1,) + d.shape, dtype=torch.uint8, device=cuda_dev)
    out = device.adaptive_points(torch.from_numpy(d).to(cuda_dev), r, StarConfig(**cfg), mask=mask)
    m = mask[0].cpu().numpy().astype(bool)
    assert np.array_equal(m, ok_ref)
    assert max_angle_deg(out[0].cpu().numpy()[m][:, 3:], n_ref[m]) < 1e-4


@pytest.mark.parametrize("shared", [False, True])
@pytest.mark.parametrize("t", [0.25, 0.5, 0.75])
def test_adaptive_cd_exact_ties(cuda_dev, shared, t):
    """Depths fx*b/d on a few exact values, so CD ranges hit t * z_c exactly:
    the fp32 filter must hand every tie to the exact walk (masks and normals
    vs the oracle's fp64 decisions)."""
    from oracle import stereonorm_oracle as orc
    from paper_2504_15121_b200 import StarConfig, StereoRig, device
    rng = np.random.default_rng(int(t * 100) + shared)
    d = rng.choice(np.array([1.0, 2.0, 4.0, 5.0, 8.0, 10.0], np.float32), (64, 72))
    d[rng.random(d.shape) < 0.02] = np.nan
    rig = StereoRig(100.0, 100.0, 35.5, 31.5, 1.0)
    cfg = dict(stop="cd", threshold=t, shared_range=shared, max_steps=6, directions=8)
    n_ref, ok_ref = orc.estimate_normals_adaptive(d.astype(np.float64),
                                                  orc.Rig(100.0, 100.0, 35.5, 31.5, 1.0),
                                                  orc.Star(**cfg))
    mask = torch.empty((1,) + d.shape, dtype=torch.uint8, device=cuda_dev)
    out = device.adaptive_points(torch.from_numpy(d).to(cuda_dev), rig, StarConfig(**cfg),
                                 mask=mask)
    m = mask[0].cpu().numpy().astype(bool)
    assert np.array_equal(m, ok_ref)
    assert max_angle_deg(out[0].cpu().numpy()[m][:, 3:], n_ref[m]) < 1e-4


def test_adaptive_random_configs_vs_oracle(cuda_dev):
    """12 random small frames x star configurations (M = 3..16 directions,
    s = 1..12 steps, ST / CD, shared range, thresholds), holes and border
    pixels: masks bit-exact and normals within 1e-4 deg of the oracle."""
    from oracle import stereonorm_oracle as orc
    from paper_2504_15121_b200 import StarConfig, StereoRig, device
    rng = np.random.default_rng(77)
    for case in range(12):
        H, W = int(rng.integers(8, 48)), int(rng.integers(8, 64))
        v, u = np.mgrid[0:H, 0:W].astype(float)
        d = 20.0 + 0.3 * u - 0.2 * v + rng.normal(0, 0.4, (H, W))
        d[rng.random((H, W)) < 0.03] = np.nan
        d = d.astype(np.float32)
        stop = str(rng.choice(["st", "cd"]))
        cfg = dict(stop=stop, threshold=float(rng.choice([0.05, 0.1, 0.3, 1.0])),
                   max_steps=int(rng.integers(1, 13)), directions=int(rng.integers(3, 17)),
                   shared_range=bool(rng.integers(0, 2)) if stop == "cd" else False)
        rig = StereoRig(300.0, 310.0, W / 2.0, H / 2.0, 0.25)
        n_ref, ok_ref = orc.estimate_normals_adaptive(d.astype(np.float64),
                                                      orc.Rig(300.0, 310.0, W / 2.0, H / 2.0, 0.25),
                                                      orc.Star(**cfg))
        mask = torch.empty((1, H, W), dtype=torch.uint8, device=cuda_dev)
        out = device.adaptive_points(torch.from_numpy(d).to(cuda_dev), rig, StarConfig(**cfg),
                                     mask=mask)
        m = mask[0].cpu().numpy().astype(bool)
        assert np.array_equal(m, ok_ref), (case, cfg)
        assert max_angle_deg(out[0].cpu().numpy()[m][:, 3:], n_ref[m]) < 1e-4, (case, cfg)


@pytest.mark.parametrize("stop", ["st", "cd"])
def test_adaptive_dynamic_spans_match_single_frames(cuda_dev, stop):
    """A batch with more 32-pixel spans than resident warps (the counter hands
    out the rest) gives every frame the records and mask of the frame run
    alone (which the static first wave covers)."""
    from paper_2504_15121_b200 import StarConfig, device, scenes
    sc = scenes.street_scene(2048, 1024)
    base = scenes.raycast(sc)[0]
    d = np.stack([scenes.add_gaussian_noise(base, 0.2, 40 + i) for i in range(3)]).astype(np.float32)
    dt = torch.from_numpy(d).to(cuda_dev)
    cfg = StarConfig(stop=stop, threshold=0.2 if stop == "st" else 0.1)
    m = torch.empty(dt.shape, dtype=torch.uint8, device=cuda_dev)
    rec = device.adaptive_points(dt, sc.rig, cfg, mask=m)
    for i in range(3):
        mi = torch.empty((1,) + dt.shape[1:], dtype=torch.uint8, device=cuda_dev)
        ri = device.adaptive_points(dt[i:i + 1], sc.rig, cfg, mask=mi)
        assert torch.equal(mi[0], m[i]), i
        assert torch.equal(ri[0].view(torch.int32), rec[i].view(torch.int32)), i
