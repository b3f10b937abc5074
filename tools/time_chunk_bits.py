"""Fused pass + bits kernel (device.oriented_points_bits) over B C3 frames in
one call vs in chunks of C frames (the bits kernel re-reads the disparities the
fused pass just read: in L2 when the chunk fits), CUDA events."""
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
out = torch.empty(B, H, W, 6, device="cuda")
bits = torch.empty(B, H, device.bit_words(W), dtype=torch.int32, device="cuda")


def run(C):
    for f0 in range(0, B, C):
        sl = slice(f0, min(B, f0 + C))
        device.oriented_points_bits(d[sl], sc.rig, 9, 0.2, out=out[sl], bits=bits[sl])


for C in (B, 64, 32, 16, 8, 4):
    for _ in range(2):
        run(C)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(3):
        run(C)
    e1.record()
    torch.cuda.synchronize()
    print(f"chunks of {C:4d}: {e0.elapsed_time(e1) * 1e3 / 3 / B:.2f} us/frame (fused + bits)")
