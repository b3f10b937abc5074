"""Concurrency, multi-device and host-path contracts of the C ABI
(include/sn_b200.h): the scratch-taking entry points on concurrent streams,
two plans on two devices in one process, pinned vs pageable host buffers,
and repeat-determinism of the racy-by-design labeller (atomicMin union-find,
sn_ccl.cu) -- the pool closes compute-sanitizer (profiles/sanitizer_r2/), so
races are hunted by repetition against a fixed answer instead."""

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _frames(n, w=512, h=256, sigma=1.0):
    from paper_2504_15121_b200 import scenes
    sc = scenes.street_scene(w, h)
    base = scenes.raycast(sc)[0]
    return np.stack([scenes.add_gaussian_noise(base, sigma, i) for i in range(n)]).astype(
        np.float32), sc.rig


def test_scratch_entry_points_on_concurrent_streams(cuda_dev):
    """sn_ccl_labels / sn_pipeline take stream-ordered scratch from the
    library's pool: two streams running them at once must not share it."""
    from paper_2504_15121_b200 import _native, device
    from paper_2504_15121_b200.kernels import KernelSpec
    d, rig = _frames(6)
    dt = torch.from_numpy(d).to(cuda_dev)
    want = device.component_labels(dt, rig, 0.2)
    want_p, want_l = device.pipeline(dt, rig, 9, 0.2)
    torch.cuda.synchronize()
    lib = _native.load()
    plan = _native.plan(cuda_dev.index)
    rs = _native.rig_struct(rig)
    off = _native.offsets_array(KernelSpec.square(9).offsets)
    streams = [torch.cuda.Stream(cuda_dev) for _ in range(2)]
    outs = []
    for rep in range(4):
        for s in streams:
            lab = torch.empty_like(want)
            pts = torch.empty_like(want_p)
            lab2 = torch.empty_like(want)
            with torch.cuda.stream(s):
                sp = ctypes.c_void_p(s.cuda_stream)
                B, H, W = dt.shape
                _native.check(lib.sn_ccl_labels(plan, dt.data_ptr(), B, H, W, ctypes.byref(rs),
                                                0.2, 0, lab.data_ptr(), sp))
                _native.check(lib.sn_pipeline(plan, dt.data_ptr(), B, H, W, ctypes.byref(rs),
                                              off.ctypes.data, len(off), 0.2, pts.data_ptr(),
                                              None, lab2.data_ptr(), sp))
            outs.append((lab, pts, lab2))
    torch.cuda.synchronize()
    for lab, pts, lab2 in outs:
        assert torch.equal(lab, want)
        assert torch.equal(lab2, want_l)
        assert torch.equal(torch.nan_to_num(pts, 7.0), torch.nan_to_num(want_p, 7.0))


def test_half_batches_on_concurrent_streams(cuda_dev):
    """From 128 frames on, sn_ccl_labels runs its second half on the plan's
    second stream: two caller streams on one plan (their second halves queue
    on that stream) must both get the one-stream answer."""
    from paper_2504_15121_b200 import _native, device
    d, rig = _frames(4, w=256, h=128)
    d = np.concatenate([d] * 33)[:130]  # 130 frames -> halves of 65
    dt = torch.from_numpy(np.ascontiguousarray(d)).to(cuda_dev)
    want = torch.stack([device.component_labels(dt[i:i + 1], rig, 0.2)[0] for i in range(4)])
    lib = _native.load()
    plan = _native.plan(cuda_dev.index)
    rs = _native.rig_struct(rig)
    streams = [torch.cuda.Stream(cuda_dev) for _ in range(2)]
    outs = []
    torch.cuda.synchronize()
    for rep in range(3):
        for s in streams:
            lab = torch.empty(dt.shape, dtype=torch.int32, device=cuda_dev)
            with torch.cuda.stream(s):
                B, H, W = dt.shape
                _native.check(lib.sn_ccl_labels(plan, dt.data_ptr(), B, H, W, ctypes.byref(rs), 0.2,
                                                0, lab.data_ptr(), ctypes.c_void_p(s.cuda_stream)))
            outs.append(lab)
    torch.cuda.synchronize()
    for lab in outs:
        for i in range(dt.shape[0]):
            assert torch.equal(lab[i], want[i % 4]), i


def test_labeller_repeat_determinism(cuda_dev):
    """The union-find's atomics race by design; its answer may not depend on
    scheduling.  50 runs of C4-style frames, each against the first."""
    from paper_2504_15121_b200 import device
    d, rig = _frames(8, 1024, 512, 1.0)
    dt = torch.from_numpy(d).to(cuda_dev)
    bits = device.passable_bits(dt, rig, 0.2)
    first = device.labels_from_bits(bits, 1024)
    for _ in range(50):
        assert torch.equal(device.labels_from_bits(bits, 1024), first)


def test_two_plans_two_devices():
    """One process, plans on two devices: per-device kernel attributes (the
    >48 KB shared-memory kernels) and per-device scratch pools."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    from paper_2504_15121_b200 import device
    d, rig = _frames(2)
    res = []
    for i in range(2):
        dev = torch.device("cuda", i)
        with torch.cuda.device(dev):
            dt = torch.from_numpy(d).to(dev)
            p, lab = device.pipeline(dt, rig, 9, 0.2)
            a = device.adaptive_points(dt, rig, __import__(
                "paper_2504_15121_b200").StarConfig(stop="st", threshold=0.5))
            res.append((p.cpu(), lab.cpu(), a.cpu()))
    for x, y in zip(res[0], res[1]):
        assert torch.equal(torch.nan_to_num(x, 7.0), torch.nan_to_num(y, 7.0))


@pytest.mark.parametrize("pinned", [True, False])
def test_host_pipeline_pinned_and_pageable(cuda_dev, pinned):
    """sn_pipeline_host copies page-locked buffers directly and stages
    pageable ones through the plan's pinned slots: same results either way,
    across several chunks (whole frames of 16 Mpx per chunk)."""
    from paper_2504_15121_b200 import _native, device
    from paper_2504_15121_b200.kernels import KernelSpec
    d, rig = _frames(5, 2048, 2048, 0.5)  # 4 Mpx frames: 4 per chunk, 2 chunks
    dt = torch.from_numpy(d).to(cuda_dev)
    want_p, want_l = device.pipeline(dt, rig, 9, 0.2)
    B, H, W = d.shape
    if pinned:
        hin = torch.from_numpy(d).pin_memory()
        hp = torch.empty((B, H, W, 6), dtype=torch.float32).pin_memory()
        hl = torch.empty((B, H, W), dtype=torch.int32).pin_memory()
        hm = torch.empty((B, H, W), dtype=torch.uint8).pin_memory()
        ptrs = (hin.data_ptr(), hp.data_ptr(), hm.data_ptr(), hl.data_ptr())
        views = (hp.numpy(), hm.numpy(), hl.numpy())
    else:
        hin = np.ascontiguousarray(d)
        hp = np.empty((B, H, W, 6), np.float32)
        hl = np.empty((B, H, W), np.int32)
        hm = np.empty((B, H, W), np.uint8)
        ptrs = (hin.ctypes.data, hp.ctypes.data, hm.ctypes.data, hl.ctypes.data)
        views = (hp, hm, hl)
    off = _native.offsets_array(KernelSpec.square(9).offsets)
    rs = _native.rig_struct(rig)
    rc = _native.load().sn_pipeline_host(_native.plan(cuda_dev.index), ptrs[0], B, H, W,
                                         ctypes.byref(rs), off.ctypes.data, len(off), 0.2,
                                         ptrs[1], ptrs[2], ptrs[3])
    _native.check(rc)
    mask = torch.empty((B, H, W), dtype=torch.uint8, device=cuda_dev)
    device.oriented_points(dt, rig, 9, mask=mask)
    assert np.array_equal(np.nan_to_num(views[0], nan=7.0),
                          np.nan_to_num(want_p.cpu().numpy(), nan=7.0))
    assert np.array_equal(views[1], mask.cpu().numpy())
    assert np.array_equal(views[2], want_l.cpu().numpy())
