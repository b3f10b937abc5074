"""Probe: the passable-bits kernel on a second stream beside the fused pass.

(Needs passable_bits_kernel built with 128-thread blocks, __launch_bounds__(128, 8);
the product keeps 256.)  The fused pass holds 2 CTAs/SM (all but ~3 KB of shared memory, ~56k of the
64k registers) and issues at ~50% of peak; a 4-warp bits block fits beside
it.  Times, on 64 C3 frames: fused alone, bits alone, both serial on one
stream, and fused (launched first) with bits on a side stream.

    python tools/overlap_bits.py [frames]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_15121_b200 import device, scenes  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
sc = scenes.street_scene(2048, 1024)
clean = torch.from_numpy(scenes.raycast(sc)[0].astype(np.float32)).cuda()
d = clean.expand(B, -1, -1).contiguous() + 0.2 * torch.randn(B, 1024, 2048, device="cuda")
out = torch.empty(B, 1024, 2048, 6, device="cuda")
bits = torch.empty((B, 1024, device.bit_words(2048)), dtype=torch.int32, device="cuda")
main = torch.cuda.current_stream()
side = torch.cuda.Stream()


def fused():
    device.oriented_points(d, sc.rig, 9, out=out)


def pbits(s=None):
    if s is None:
        device.passable_bits(d, sc.rig, 0.2, bits=bits)
    else:
        with torch.cuda.stream(s):
            device.passable_bits(d, sc.rig, 0.2, bits=bits)


def both_serial():
    fused()
    pbits()


def both_overlap():
    fork = torch.cuda.Event()
    fork.record(main)
    fused()
    side.wait_event(fork)
    pbits(side)
    join = torch.cuda.Event()
    join.record(side)
    main.wait_event(join)


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(main)
    for _ in range(n):
        fn()
    e1.record(main)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n / B


ref = bits.clone()
pbits()
torch.cuda.synchronize()
ref.copy_(bits)
for name, fn in [("fused", fused), ("bits", pbits), ("serial", both_serial),
                 ("overlap", both_overlap), ("serial", both_serial), ("overlap", both_overlap)]:
    print(f"{name:8s} {timeit(fn):7.2f} us/frame")
bits.zero_()
both_overlap()
torch.cuda.synchronize()
print("bits identical after overlap:", bool(torch.equal(bits, ref)))
