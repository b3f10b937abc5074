"""Predicate + labels from disparity (device.component_labels: bits kernel +
tile / seam / resolve) at C3, us/frame over B-frame batches (CUDA events)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_15121_b200 import device, scenes  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
torch.manual_seed(0)
sc = scenes.street_scene(2048, 1024)
base = torch.from_numpy(scenes.raycast(sc)[0].astype(np.float32)).cuda()
d = base.expand(B, -1, -1).contiguous() + 0.2 * torch.randn(B, 1024, 2048, device="cuda")
ws = device.ccl_workspace(B, 1024, 2048, d.device)
lab = torch.empty(B, 1024, 2048, dtype=torch.int32, device="cuda")
for t in (0.05, 0.2, 1.0):
    def run():
        device.component_labels(d, sc.rig, t, out=lab, workspace=ws)
    for _ in range(2):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    n = 5
    e0.record()
    for _ in range(n):
        run()
    e1.record()
    torch.cuda.synchronize()
    h = int(torch.sum(lab[:, ::7, ::5].to(torch.int64) % 1000003))
    print(json.dumps({"t": t, "us_per_frame": round(e0.elapsed_time(e1) * 1e3 / n / B, 2),
                      "hash": h}), flush=True)
