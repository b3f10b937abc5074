"""Tile-pass time per frame alone (the labeller's first kernel) on C3 bit masks,
for compile-time variants of it (exp/*.so via SN_B200_LIB)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_15121_b200 import device, scenes  # noqa: E402

B = 64
sc = scenes.street_scene(2048, 1024)
base = torch.from_numpy(scenes.raycast(sc)[0].astype(np.float32)).cuda()
d = base.expand(B, -1, -1).contiguous() + 0.2 * torch.randn(B, 1024, 2048, device="cuda")
ws = device.ccl_workspace(B, 1024, 2048, d.device)
lab = torch.empty(B, 1024, 2048, dtype=torch.int32, device="cuda")
for t in (0.05, 0.2, 1.0):
    bits = device.passable_bits(d, sc.rig, t)
    for _ in range(2):
        device.labels_from_bits(bits, 2048, out=lab, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(5):
        device.labels_from_bits(bits, 2048, out=lab, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    print(json.dumps({"t": t, "labels_us_per_frame": round(e0.elapsed_time(e1) * 1e3 / 5 / B, 2)}))
