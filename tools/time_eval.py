"""Time the device accuracy evaluation at C3 frame size:
angle map + per-frame stats from the fused pass's records vs fp64 ground
truth, and summarize of a given fp64 map.  CUDA events, inputs >> L2."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_15121_b200 import KernelSpec, device, scenes  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
H, W = 1024, 2048
sc = scenes.street_scene(W, H)
d0, _, n0 = scenes.raycast(sc)
gt = torch.from_numpy(np.ascontiguousarray(n0, dtype=np.float64)).cuda().expand(B, -1, -1, -1).contiguous()
gm = torch.isfinite(gt).all(-1).to(torch.uint8)
d = torch.from_numpy(d0.astype(np.float32)).cuda().expand(B, -1, -1).contiguous()
d += 0.2 * torch.randn_like(d)
rec = device.oriented_points(d, sc.rig, KernelSpec.square(9))


def timed(fn, n=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


for name, fn in [("angular_error+map", lambda: device.angular_error(rec, gt, gm)),
                 ("angular_error(stats only)", lambda: device.angular_error(rec, gt, gm, want_map=False))]:
    ms = timed(fn)
    print(json.dumps({"kernel": name, "us_per_frame": round(ms * 1e3 / B, 2),
                      "mpx_per_s": round(H * W * B / ms / 1e3, 1)}), flush=True)
err, _ = device.angular_error(rec, gt, gm)
ms = timed(lambda: device.error_stats(err))
print(json.dumps({"kernel": "error_stats", "us_per_frame": round(ms * 1e3 / B, 2),
                  "mpx_per_s": round(H * W * B / ms / 1e3, 1)}), flush=True)
