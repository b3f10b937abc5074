"""Time the adaptive star-fill pass at C3 (2048x1024) for a few configs."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2504_15121_b200 import StarConfig, device, scenes

sc = scenes.street_scene(2048, 1024)
clean = torch.from_numpy(scenes.raycast(sc)[0].astype(np.float32)).cuda()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
d = clean.expand(B, -1, -1).contiguous() + 0.2 * torch.randn(B, 1024, 2048, device="cuda")
out = torch.empty(B, 1024, 2048, 6, device="cuda")
for cfg in [dict(stop="cd", threshold=0.1), dict(stop="st", threshold=0.2),
            dict(stop="cd", threshold=0.1, max_steps=30, directions=16),
            dict(stop="st", threshold=0.2, max_steps=30, directions=16)]:
    c = StarConfig(**cfg)
    for _ in range(2):
        device.adaptive_points(d, sc.rig, c, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    n = 5
    for _ in range(n):
        device.adaptive_points(d, sc.rig, c, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n / B
    print(f"{cfg}: {ms * 1e3:8.1f} us/frame  {2048 * 1024 / ms / 1e3:8.0f} Mpx/s")
