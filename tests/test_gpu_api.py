"""The C ABI's error contract and concurrency on the device:
invalid arguments -> SN_EINVAL (ValueError), collinear patterns ->
SN_EDEGENERATE (DegenerateSupportError), empty batches are no-ops, and calls
from several host threads on their own streams / workspaces give the same
results as sequential calls (the reference is safe to call concurrently,
SPEC.md:97-98)."""

import ctypes
import threading

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _lib_plan(dev):
    from paper_2504_15121_b200 import _native
    return _native.load(), _native.plan(dev.index)


def test_abi_error_codes(cuda_dev):
    from paper_2504_15121_b200 import _native, StereoRig
    lib, plan = _lib_plan(cuda_dev)
    d = torch.ones((1, 16, 32), device=cuda_dev)
    out = torch.empty((1, 16, 32, 6), device=cuda_dev)
    rs = _native.rig_struct(StereoRig(100.0, 100.0, 16.0, 8.0, 0.2))
    sq = np.array([[dx, dy] for dy in (-1, 0, 1) for dx in (-1, 0, 1)], np.int32)
    call = lambda *a: lib.sn_oriented_points(*a)  # noqa: E731
    ok = call(plan, d.data_ptr(), 1, 16, 32, ctypes.byref(rs), sq.ctypes.data, 9, out.data_ptr(),
              None, None)
    assert ok == 0
    # bad shapes / NULL buffers / NULL plan -> 1, with a message
    assert call(plan, d.data_ptr(), -1, 16, 32, ctypes.byref(rs), sq.ctypes.data, 9,
                out.data_ptr(), None, None) == 1
    assert lib.sn_last_error()
    assert call(plan, None, 1, 16, 32, ctypes.byref(rs), sq.ctypes.data, 9, out.data_ptr(),
                None, None) == 1
    assert call(None, d.data_ptr(), 1, 16, 32, ctypes.byref(rs), sq.ctypes.data, 9,
                out.data_ptr(), None, None) == 1
    bad = _native.rig_struct(StereoRig(100.0, 100.0, 16.0, 8.0, 0.2))
    bad.fx = -1.0
    assert call(plan, d.data_ptr(), 1, 16, 32, ctypes.byref(bad), sq.ctypes.data, 9,
                out.data_ptr(), None, None) == 1
    # collinear offsets: degenerate support (kernels.py:91-93) -> 2
    line = np.array([[-1, 0], [0, 0], [1, 0]], np.int32)
    assert call(plan, d.data_ptr(), 1, 16, 32, ctypes.byref(rs), line.ctypes.data, 3,
                out.data_ptr(), None, None) == 2
    # empty batch: nothing to do, NULL buffers allowed
    assert call(plan, None, 0, 16, 32, ctypes.byref(rs), sq.ctypes.data, 9, None, None,
                None) == 0
    torch.cuda.synchronize()


def test_python_errors_map_to_reference_exceptions(cuda_dev):
    import paper_2504_15121_b200 as sn
    from paper_2504_15121_b200 import device
    d = torch.ones((8, 8), device=cuda_dev)
    with pytest.raises(sn.DegenerateSupportError):
        device.oriented_points(d, sn.StereoRig(10.0, 10.0, 4.0, 4.0, 0.1),
                               sn.KernelSpec(np.array([[0, 0], [1, 1], [2, 2]])))
    with pytest.raises(ValueError):
        device.component_labels(d, sn.StereoRig(10.0, 10.0, 4.0, 4.0, 0.1), -1.0)
    with pytest.raises(ValueError):
        device.oriented_points(d.double().int(), sn.StereoRig(10.0, 10.0, 4.0, 4.0, 0.1), 3)


def test_concurrent_host_threads(cuda_dev):
    """4 host threads, each with its own stream and workspace, run the whole
    pipeline on different batches at the same time; every result equals the
    sequential one."""
    from paper_2504_15121_b200 import device, scenes
    sc = scenes.street_scene(512, 256)
    clean = scenes.raycast(sc)[0]
    batches = [torch.from_numpy(np.stack([scenes.add_gaussian_noise(clean, 0.3, 10 * i + j)
                                          for j in range(3)]).astype(np.float32)).to(cuda_dev)
               for i in range(4)]
    ref = [device.pipeline(b, sc.rig, 9, 0.2) for b in batches]
    torch.cuda.synchronize()
    got = [None] * 4
    errors = []

    def work(i):
        try:
            s = torch.cuda.Stream(cuda_dev)
            with torch.cuda.stream(s):
                ws = device.ccl_workspace(3, 256, 512, cuda_dev)
                for _ in range(3):
                    got[i] = device.pipeline(batches[i], sc.rig, 9, 0.2, workspace=ws)
            s.synchronize()
        except Exception as exc:  # pragma: no cover - reported below
            errors.append(exc)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors
    for (p0, l0), (p1, l1) in zip(ref, got):
        assert torch.equal(torch.nan_to_num(p0, 7.0), torch.nan_to_num(p1, 7.0))
        assert torch.equal(l0, l1)


def test_cuda_graph_capture(cuda_dev):
    """The device pipeline is stream-ordered with no host synchronisation, so it
    can be captured once into a CUDA graph and replayed (small frames: the five
    launches become one graph launch); replays match eager calls."""
    from paper_2504_15121_b200 import device, scenes
    sc = scenes.street_scene(640, 480)
    clean = scenes.raycast(sc)[0]
    d = torch.from_numpy(scenes.add_gaussian_noise(clean, 0.2, 1).astype(np.float32)).to(cuda_dev)
    d = d[None].contiguous()
    out = torch.empty((1, 480, 640, 6), device=cuda_dev)
    lab = torch.empty((1, 480, 640), dtype=torch.int32, device=cuda_dev)
    ws = device.ccl_workspace(1, 480, 640, cuda_dev)
    s = torch.cuda.Stream(cuda_dev)
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm-up outside capture (one-time attribute setup)
        device.pipeline(d, sc.rig, 9, 0.2, out=out, labels=lab, workspace=ws)
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        device.pipeline(d, sc.rig, 9, 0.2, out=out, labels=lab, workspace=ws)
    ref_out, ref_lab = device.pipeline(d, sc.rig, 9, 0.2)
    for seed in (2, 3):
        d.copy_(torch.from_numpy(scenes.add_gaussian_noise(clean, 0.2, seed).astype(np.float32))
                .to(cuda_dev)[None])
        g.replay()
        ref_out, ref_lab = device.pipeline(d, sc.rig, 9, 0.2)
        torch.cuda.synchronize()
        assert torch.equal(torch.nan_to_num(out, 7.0), torch.nan_to_num(ref_out, 7.0))
        assert torch.equal(lab, ref_lab)


def test_batch_beyond_int32_pixels(cuda_dev):
    """A batch of more than 2^31 pixels (70,000 frames of 256x128: 9.2 GB in,
    55 GB of records out) through one fused-pass call: 64-bit batch offsets
    and 3D TMA coordinates past 2^16 frames -- the first, a middle and the
    last frames equal the same frames processed alone."""
    from paper_2504_15121_b200 import device, scenes
    free, _ = torch.cuda.mem_get_info(cuda_dev)
    B, H, W = 70000, 128, 256
    if free < 70 * 2**30:
        pytest.skip("needs ~70 GB of free device memory")
    sc = scenes.street_scene(W, H)
    base = torch.from_numpy(scenes.raycast(sc)[0].astype(np.float32)).to(cuda_dev)
    d = base.expand(B, -1, -1).contiguous()
    d[:, 10, :] += torch.arange(B, device=cuda_dev, dtype=torch.float32)[:, None] * 1e-3
    out = device.oriented_points(d, sc.rig, 9)
    for i in (0, 35001, B - 1):
        one = device.oriented_points(d[i], sc.rig, 9)[0]
        assert torch.equal(torch.nan_to_num(out[i], 7.0), torch.nan_to_num(one, 7.0)), i
    del out
    torch.cuda.empty_cache()
    # labels: more frames than one launch's grid holds (65535), chunked inside
    lab = device.component_labels(d, sc.rig, 0.2)
    for i in (0, 65534, 65535, B - 1):
        assert torch.equal(lab[i], device.component_labels(d[i], sc.rig, 0.2)[0]), i
    del lab, d
    torch.cuda.empty_cache()


@pytest.mark.parametrize("shape", [(0, 16, 32), (2, 0, 32), (2, 16, 0)])
def test_empty_inputs(cuda_dev, shape):
    """Empty batches / frames through every device entry point: correctly
    shaped empty results, no error, no launch on zero pixels."""
    from paper_2504_15121_b200 import StarConfig, StereoRig, device
    rig = StereoRig(100.0, 100.0, 8.0, 8.0, 0.2)
    d = torch.empty(shape, device=cuda_dev)
    B, H, W = shape
    assert device.oriented_points(d, rig, 3).shape == (B, H, W, 6)
    assert device.passable_bits(d, rig, 0.2).shape == (B, H, device.bit_words(W))
    assert device.component_labels(d, rig, 0.2).shape == (B, H, W)
    pts, lab = device.pipeline(d, rig, 3, 0.2)
    assert pts.shape == (B, H, W, 6) and lab.shape == (B, H, W)
    assert device.adaptive_points(d, rig, StarConfig(stop="cd", threshold=0.1)).shape == (B, H, W, 6)
    m = torch.zeros(shape, dtype=torch.uint8, device=cuda_dev)
    cloud, offs = device.compact_cloud(pts, m)
    assert cloud.shape == (0, 6) and offs.shape == (B + 1,) and int(offs[-1]) == 0
    raw = torch.from_numpy(np.zeros(shape, np.uint16)).to(cuda_dev)
    assert device.dequant_png16(raw, 256.0, 0).shape == (B, H, W)
    torch.cuda.synchronize()


@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("crop", [(0, 512), (3, 300), (4, 260)])
def test_row_pitched_input(cuda_dev, dtype, crop):
    """sn_oriented_points_strided: a column crop of wider frames (row pitch
    ld > W; 16-byte-aligned pitches go to TMA directly, others through a
    packed copy) gives the records of the same frames made contiguous."""
    import torch
    from paper_2504_15121_b200 import device, scenes
    sc = scenes.street_scene(600, 96)
    d = np.stack([scenes.add_gaussian_noise(scenes.raycast(sc)[0], 0.3, s) for s in (1, 2)])
    full = torch.from_numpy(d).to(cuda_dev, dtype=getattr(torch, dtype))
    c0, c1 = crop
    view = full[:, :, c0:c1]
    assert not view.is_contiguous()
    m1 = torch.empty(view.shape, dtype=torch.uint8, device=cuda_dev)
    m2 = torch.empty(view.shape, dtype=torch.uint8, device=cuda_dev)
    a = device.oriented_points(view, sc.rig, 9, mask=m1)
    b = device.oriented_points(view.contiguous(), sc.rig, 9, mask=m2)
    assert torch.equal(m1, m2)
    assert torch.equal(torch.nan_to_num(a, 7.0), torch.nan_to_num(b, 7.0))
