"""Fused-pass time per frame vs batch size (C3 2048x1024 and C2 2888x1920
frames), CUDA events, L2 flushed (256 MB read) before each repetition."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_15121_b200 import device, scenes  # noqa: E402

flush = torch.ones(64 << 20, device="cuda")
sink = torch.empty((), device="cuda")
res = {}
for name, sc in (("C3", scenes.street_scene(2048, 1024)), ("C2", scenes.sphere_scene(2888, 1920))):
    base = torch.from_numpy(np.nan_to_num(scenes.raycast(sc)[0], nan=10.0).astype(np.float32)).cuda()
    for B in (1, 2, 4, 16, 64):
        if name == "C2" and B > 16:
            continue
        d = base.expand(B, -1, -1).contiguous() + 0.2 * torch.randn(B, *base.shape, device="cuda")
        out = torch.empty(*d.shape, 6, device="cuda")
        device.oriented_points(d, sc.rig, 9, out=out)
        tot = 0.0
        for _ in range(5):
            sink.copy_(flush.sum())
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            device.oriented_points(d, sc.rig, 9, out=out)
            e1.record()
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        us = tot / 5 * 1e3 / B
        px = base.numel()
        res[f"{name}_B{B}"] = {"us_per_frame": round(us, 2),
                               "frac_hbm": round(28 * px / (us * 1e-6) / 1e9 / 6535.1, 3)}
print(json.dumps(res))
