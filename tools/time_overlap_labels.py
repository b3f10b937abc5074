"""Labeller overlap probe (C3, t = 0.2): bits + labels of B frames as one batch
on one stream, vs frame chunks alternating over 2 (or 3) streams, so that the
issue-bound tile pass of one chunk runs beside the memory-bound bits / resolve
kernels of another.  CUDA events on the default stream around all of it."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_15121_b200 import device, scenes  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
torch.manual_seed(0)
H, W = 1024, 2048
sc = scenes.street_scene(W, H)
base = torch.from_numpy(scenes.raycast(sc)[0].astype(np.float32)).cuda()
d = base.expand(B, -1, -1).contiguous() + 0.2 * torch.randn(B, H, W, device="cuda")
lab = torch.empty(B, H, W, dtype=torch.int32, device="cuda")
bits = torch.empty(B, H, device.bit_words(W), dtype=torch.int32, device="cuda")
ws_all = device.ccl_workspace(B, H, W, d.device)


def whole():
    device.passable_bits(d, sc.rig, 0.2, bits=bits)
    device.labels_from_bits(bits, W, out=lab, workspace=ws_all)


def chunked(C, NS):
    streams = [torch.cuda.Stream() for _ in range(NS)]
    wss = [device.ccl_workspace(C, H, W, d.device) for _ in range(NS)]
    main = torch.cuda.current_stream()

    def run():
        for s in streams:
            s.wait_stream(main)
        for k, f0 in enumerate(range(0, B, C)):
            s = streams[k % NS]
            with torch.cuda.stream(s):
                sl = slice(f0, min(B, f0 + C))
                device.passable_bits(d[sl], sc.rig, 0.2, bits=bits[sl])
                device.labels_from_bits(bits[sl], W, out=lab[sl], workspace=wss[k % NS])
        for s in streams:
            main.wait_stream(s)
    return run


def timeit(fn, n=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n / B


t = timeit(whole)
ref = lab.clone()
print(f"whole batch, 1 stream: {t:.2f} us/frame")
for C in (64, 32, 16):
    for NS in (2, 3):
        lab.zero_()
        t = timeit(chunked(C, NS))
        ok = torch.equal(lab, ref)
        print(f"chunks of {C}, {NS} streams: {t:.2f} us/frame  labels equal: {ok}")
