"""Time the oriented-cloud compaction at C3: records +
mask from the fused pass -> [N, 6] vertices in raster order.  Algorithmic
bytes: mask 1 B/px (read by the count and scatter passes: 2 B/px) + 24 B per
kept vertex read + 24 B per kept vertex written."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_15121_b200 import device, scenes  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
sc = scenes.street_scene(2048, 1024)
clean = torch.from_numpy(scenes.raycast(sc)[0].astype(np.float32)).cuda()
d = clean.expand(B, -1, -1).contiguous() + 0.2 * torch.randn(B, 1024, 2048, device="cuda")
mask = torch.empty(B, 1024, 2048, dtype=torch.uint8, device="cuda")
rec = device.oriented_points(d, sc.rig, 9, mask=mask)
for _ in range(2):
    cloud, offs = device.compact_cloud(rec, mask)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
n = 5
e0.record()
for _ in range(n):
    cloud, offs = device.compact_cloud(rec, mask)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
kept = int(offs[-1])
px = B * 1024 * 2048
bytes_ = 2 * px + 48 * kept
print(json.dumps({"kernel": "compact_cloud", "us_per_frame": round(ms * 1e3 / B, 2),
                  "kept_fraction": round(kept / px, 4),
                  "achieved_gbps": round(bytes_ / (ms * 1e-3) / 1e9, 1),
                  "note": "includes the host read of the vertex count (one sync per call)"}))
