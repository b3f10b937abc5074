"""Fused pass time for aligned vs unaligned widths (KITTI-like 1242x375 takes
the generic kernel when W % 4 != 0)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2504_15121_b200 import device, scenes

for W, H in ((1240, 375), (1242, 375), (1241, 375)):
    sc = scenes.street_scene(W, H)
    B = 64
    d = torch.from_numpy(scenes.raycast(sc)[0].astype(np.float32)).cuda().expand(B, -1, -1).contiguous()
    d += 0.2 * torch.randn_like(d)
    out = torch.empty(B, H, W, 6, device="cuda")
    for _ in range(2):
        device.oriented_points(d, sc.rig, 9, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        device.oriented_points(d, sc.rig, 9, out=out)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 5 / B
    print(f"{W}x{H}: {us:.2f} us/frame  {W * H / us:.0f} Mpx/s")
