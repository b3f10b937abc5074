"""Whole-step overlap probe (C3, t = 0.2, k = 9): fused pass + passable bits +
labels of B frames on one stream, vs frame chunks spread over 2 streams, with
and without a stagger (chunk c's first kernel waits for chunk c-1's fused pass,
so a chunk's issue-bound tile pass meets the next chunk's memory-bound fused
pass instead of its twin).  CUDA events on the default stream around it all;
records and labels checked equal to the one-stream run.

    python tools/time_overlap_step.py [frames]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_15121_b200 import device, scenes  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
torch.manual_seed(0)
H, W = 1024, 2048
sc = scenes.street_scene(W, H)
base = torch.from_numpy(scenes.raycast(sc)[0].astype(np.float32)).cuda()
d = base.expand(B, -1, -1).contiguous() + 0.2 * torch.randn(B, H, W, device="cuda")
out = torch.empty(B, H, W, 6, device="cuda")
lab = torch.empty(B, H, W, dtype=torch.int32, device="cuda")
bits = torch.empty(B, H, device.bit_words(W), dtype=torch.int32, device="cuda")
ws_all = device.ccl_workspace(B, H, W, d.device)


def whole():
    device.oriented_points(d, sc.rig, 9, out=out)
    device.passable_bits(d, sc.rig, 0.2, bits=bits)
    device.labels_from_bits(bits, W, out=lab, workspace=ws_all)


def chunked(C, NS, stagger):
    streams = [torch.cuda.Stream() for _ in range(NS)]
    wss = [device.ccl_workspace(C, H, W, d.device) for _ in range(NS)]
    main = torch.cuda.current_stream()

    def run():
        for s in streams:
            s.wait_stream(main)
        prev = None
        for k, f0 in enumerate(range(0, B, C)):
            s = streams[k % NS]
            sl = slice(f0, min(B, f0 + C))
            with torch.cuda.stream(s):
                if stagger and prev is not None:
                    s.wait_event(prev)
                device.oriented_points(d[sl], sc.rig, 9, out=out[sl])
                if stagger:
                    prev = torch.cuda.Event()
                    prev.record(s)
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
ref_lab = lab.clone()
ref_out = out.clone()
print(f"whole batch, 1 stream: {t:.2f} us/frame")
for C, NS, st in ((128, 2, False), (128, 2, True), (64, 2, True), (64, 3, True), (32, 2, True),
                  (32, 3, True)):
    lab.zero_()
    out.zero_()
    t = timeit(chunked(C, NS, st))
    ok = torch.equal(lab, ref_lab) and torch.equal(out.nan_to_num(), ref_out.nan_to_num())
    print(f"chunks of {C}, {NS} streams, stagger {st}: {t:.2f} us/frame  equal: {ok}")
