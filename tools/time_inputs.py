"""Fused pass time by input type at C3 (fp32, fp64, 16-bit PNG samples)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2504_15121_b200 import device, scenes

sc = scenes.street_scene(2048, 1024)
B = 32
base = torch.from_numpy(scenes.raycast(sc)[0].astype(np.float32)).cuda()
d32 = base.expand(B, -1, -1).contiguous() + 0.2 * torch.randn(B, 1024, 2048, device="cuda")
d64 = d32.double()
raw = torch.clamp(torch.round(d32 * 256 + 1), 1, 65535).to(torch.int32).to(torch.uint16)
out = torch.empty(B, 1024, 2048, 6, device="cuda")


def t(fn, n=5):
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


print("fp32 ", round(t(lambda: device.oriented_points(d32, sc.rig, 9, out=out)), 2), "us/frame")
print("fp64 ", round(t(lambda: device.oriented_points(d64, sc.rig, 9, out=out)), 2), "us/frame")
print("png16", round(t(lambda: device.oriented_points_png16(raw, sc.rig, 9, out=out)), 2), "us/frame")
