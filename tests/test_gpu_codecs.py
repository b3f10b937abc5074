"""Device input codecs vs the reference readers.

Bars: decoded PFM samples bit-exact (NaN pattern included); dequantised
PNG16 disparities bit-exact in fp64 and equal to that value rounded once in
fp32; the fused PNG16 pass (2 B/px read) meets the fused pass's own bars
against estimate_normals_fixed + triangulate_grid on the reference's decoded
field: normal masks bit-exact, normals within 1e-4 deg, points within 1e-5
relative.  Goldens: tests/golden/make_golden_codecs.py.
"""

import numpy as np
import pytest
import torch

from helpers import rig_of
from test_gpu_parity import _check_record

pytestmark = pytest.mark.gpu


def _bits_equal(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


def test_pfm_golden(codec_golden, cuda_dev):
    from paper_2504_15121_b200 import formats
    for name, c in codec_golden["pfm"].items():
        data = bytes(c["bytes"])
        ch = int(c["channels"])
        magic = b"PF" if ch == 3 else b"Pf"
        t = formats.read_pfm_device(data, magic, device=cuda_dev)
        torch.cuda.synchronize()
        got = t.cpu().numpy()
        # the file's own float32 samples, top row first
        _, w, h, scale, pos = formats._pfm_header(data)
        shape = (h, w, 3) if ch == 3 else (h, w)
        want = np.frombuffer(data[pos:], ">f4" if scale > 0 else "<f4").reshape(shape)[::-1]
        assert _bits_equal(got, want.astype("=f4")), name
        field = formats.read_pfm_normals(data) if ch == 3 else formats.read_pfm(data)
        vals = field.vectors if ch == 3 else field.values
        assert np.array_equal(field.mask, c["mask"]), name
        assert np.array_equal(vals, c["values"], equal_nan=True), name


@pytest.mark.parametrize("B,H,W,ch,be", [(3, 17, 64, 1, True), (2, 5, 12, 3, False),
                                         (1, 9, 7, 1, False), (4, 33, 40, 3, True)])
def test_decode_pfm_batched(cuda_dev, B, H, W, ch, be):
    from paper_2504_15121_b200 import device
    rng = np.random.default_rng(B * 100 + W)
    shape = (B, H, W, 3) if ch == 3 else (B, H, W)
    g = rng.normal(0, 100, shape).astype(np.float32)
    g.reshape(-1)[::13] = np.nan
    payload = np.ascontiguousarray(g[:, ::-1]).astype(">f4" if be else "<f4")
    t = torch.from_numpy(np.frombuffer(payload.tobytes(), np.uint8).copy()).to(cuda_dev)
    out = device.decode_pfm(t, H, W, ch, big_endian=be)
    torch.cuda.synchronize()
    assert _bits_equal(out.cpu().numpy(), g)


def test_png16_golden(codec_golden, cuda_dev):
    from paper_2504_15121_b200 import device, formats
    for name, c in codec_golden["png"].items():
        data = bytes(c["bytes"])
        scale, inv = float(c["scale"]), int(c["invalid"])
        d64 = formats.read_disparity_png16_device(data, scale, inv, dtype=torch.float64,
                                                  device=cuda_dev).cpu().numpy()
        assert _bits_equal(d64, c["values"]), name
        d32 = formats.read_disparity_png16_device(data, scale, inv, device=cuda_dev)
        assert _bits_equal(d32.cpu().numpy(), c["values"].astype(np.float32)), name
        f = formats.read_disparity_png16(data, scale, inv)
        assert np.array_equal(f.mask, c["mask"]), name
        assert _bits_equal(f.values, c["values"]), name
        # both dtypes from one call
        raw = torch.from_numpy(c["raw"]).to(cuda_dev)
        if 0 <= inv <= 0xFFFF:
            o = device.dequant_png16(raw, scale, inv)
            assert _bits_equal(o[0].cpu().numpy(), c["values"]), name


@pytest.mark.parametrize("shape", [(2, 64, 64), (1, 3, 5), (3, 16, 24)])
def test_dequant_paths(cuda_dev, shape):
    """16-byte vector path (n % 8 == 0) and the scalar tail path."""
    from paper_2504_15121_b200 import device
    rng = np.random.default_rng(sum(shape))
    raw = rng.integers(0, 65536, shape).astype(np.uint16)
    for scale, inv in [(256.0, 0), (7.3, 65535), (-0.5, None)]:
        want = (raw.astype(np.float64) - 1.0) / scale
        if inv is not None:
            want[raw == inv] = np.nan
        got = device.dequant_png16(torch.from_numpy(raw).to(cuda_dev), scale, inv)
        assert _bits_equal(got.cpu().numpy(), want)
        got32 = device.dequant_png16(torch.from_numpy(raw).to(cuda_dev), scale, inv,
                                     dtype=torch.float32)
        assert _bits_equal(got32.cpu().numpy(), want.astype(np.float32))


@pytest.mark.parametrize("name", ["street_s256_k9", "street_s100_k5", "street_s256_k15"])
def test_oriented_points_png16_golden(codec_golden, cuda_dev, name):
    from paper_2504_15121_b200 import KernelSpec, device, formats
    c = codec_golden["fused"][name]
    raw = formats.read_png16_raw_device(bytes(c["bytes"]), device=cuda_dev)
    k = int(c["k"])
    mask = torch.empty((1,) + tuple(raw.shape), dtype=torch.uint8, device=cuda_dev)
    out = device.oriented_points_png16(raw, rig_of(c["rig"]), KernelSpec.square(k),
                                       scale=float(c["scale"]), invalid_value=0, mask=mask)
    torch.cuda.synchronize()
    _check_record(out[0].cpu().numpy(), mask[0].cpu().numpy(), c)
    # same records as the fp64 path on the dequantised field up to fp32 rounding of d
    d64 = device.dequant_png16(raw, float(c["scale"]), 0)
    ref = device.oriented_points(d64, rig_of(c["rig"]), KernelSpec.square(k))
    a, b = out.cpu().numpy(), ref.cpu().numpy()
    assert np.array_equal(np.isnan(a), np.isnan(b))


@pytest.mark.parametrize("B,H,W,k", [(3, 96, 136, 7), (2, 101, 72, 9), (1, 17, 8, 3),
                                     (2, 64, 520, 17), (2, 40, 1242, 9), (1, 33, 37, 5)])
def test_oriented_points_png16_batched(cuda_dev, B, H, W, k):
    """Batches with invalid holes and ragged tiles, vs the fp32 path on the
    decoded values (power-of-two scale: dequantised values are exact in fp32)."""
    from paper_2504_15121_b200 import KernelSpec, StereoRig, device
    rng = np.random.default_rng(5 + H)
    raw = rng.integers(2000, 9000, (B, H, W)).astype(np.uint16)
    raw[rng.random(raw.shape) < 0.01] = 0
    rig = StereoRig(200.0, 210.0, 70.0, 45.0, 0.3)
    r = torch.from_numpy(raw).to(cuda_dev)
    m1 = torch.empty((B, H, W), dtype=torch.uint8, device=cuda_dev)
    m2 = torch.empty_like(m1)
    o1 = device.oriented_points_png16(r, rig, KernelSpec.square(k), scale=64.0, mask=m1)
    d = device.dequant_png16(r, 64.0, 0, dtype=torch.float32)
    o2 = device.oriented_points(d, rig, KernelSpec.square(k), mask=m2)
    torch.cuda.synchronize()
    assert torch.equal(m1, m2)
    assert _bits_equal(o1.cpu().numpy(), o2.cpu().numpy())


def test_png16_rejects(cuda_dev):
    from paper_2504_15121_b200 import KernelSpec, StereoRig, device
    rig = StereoRig(100.0, 100.0, 10.0, 10.0, 0.2)
    with pytest.raises(ValueError, match="square kernel"):
        r = torch.from_numpy(np.zeros((1, 16, 24), np.uint16)).to(cuda_dev)
        device.oriented_points_png16(r, rig, KernelSpec(np.array([[0, 0], [1, 0], [0, 1]])))
    r = torch.from_numpy(np.zeros((1, 16, 24), np.uint16)).to(cuda_dev)
    with pytest.raises(ValueError, match="scale"):
        device.oriented_points_png16(r, rig, KernelSpec.square(5), scale=0.0)
    with pytest.raises(ValueError, match="scale"):
        device.dequant_png16(r, 0.0)


def test_dequant_division_exhaustive(cuda_dev):
    """Every 16-bit sample for 40 scales (powers of two, decimals, random,
    near the 2^+-100 fast-division limits and beyond): the device's
    reciprocal-and-correct division equals numpy's correctly rounded fp64
    (raw - 1) / scale bit for bit."""
    from paper_2504_15121_b200 import device
    rng = np.random.default_rng(99)
    scales = [256.0, 100.0, 3.0, 7.3, 1.0 / 3.0, -64.0, -0.1, 65535.0, 2.0 ** -100, 2.0 ** 100,
              1.5 * 2.0 ** -101, 1.1 * 2.0 ** 100, 1e-300, 1e300]
    scales += list(rng.uniform(0.01, 1000.0, 14)) + list(np.exp(rng.uniform(-60, 60, 12)))
    raw = np.arange(65536, dtype=np.uint16).reshape(256, 256)
    t = torch.from_numpy(raw).to(cuda_dev)
    a = raw.astype(np.float64) - 1.0
    for s in scales:
        with np.errstate(over="ignore", under="ignore"):
            want = a / s
        want[raw == 0] = np.nan
        got = device.dequant_png16(t, float(s), 0).cpu().numpy()
        assert _bits_equal(got[0], want), f"scale {s!r}"
