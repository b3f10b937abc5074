"""Labeller time per frame (bits kernel + tile / seam / resolve) at C3
(sigma 0.2) and C4 (sigma 1.0 + dilated holes) for t in {0.05, 0.2, 1.0},
CUDA events over 64-frame batches; prints component counts too."""
import json
import sys

import numpy as np
import torch
from scipy import ndimage

sys.path.insert(0, ".")
from paper_2504_15121_b200 import device, scenes  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
sc = scenes.street_scene(2048, 1024)
clean = scenes.raycast(sc)[0]
base = torch.from_numpy(clean.astype(np.float32)).cuda()
for cfg in ("C3", "C4"):
    sigma = 0.2 if cfg == "C3" else 1.0
    d = base.expand(B, -1, -1).contiguous() + sigma * torch.randn(B, 1024, 2048, device="cuda")
    if cfg == "C4":
        for i in range(B):
            holes = ndimage.binary_dilation(np.random.default_rng(1000 + i).random(clean.shape) < 0.002,
                                            iterations=3)
            d[i][torch.from_numpy(holes).cuda()] = float("nan")
    ws = device.ccl_workspace(B, 1024, 2048, d.device)
    lab = torch.empty(B, 1024, 2048, dtype=torch.int32, device="cuda")
    bits = torch.empty(B, 1024, device.bit_words(2048), dtype=torch.int32, device="cuda")
    for t in (0.05, 0.2, 1.0):
        def run():
            device.passable_bits(d, sc.rig, t, bits=bits)
            device.labels_from_bits(bits, 2048, out=lab, workspace=ws)
        for _ in range(2):
            run()
        torch.cuda.synchronize()
        e0, e1, e2 = (torch.cuda.Event(True) for _ in range(3))
        n = 5
        e0.record()
        for _ in range(n):
            device.passable_bits(d, sc.rig, t, bits=bits)
        e1.record()
        for _ in range(n):
            device.labels_from_bits(bits, 2048, out=lab, workspace=ws)
        e2.record()
        torch.cuda.synchronize()
        l0 = lab[0]
        comps = int(((l0 >= 0) & (l0 == torch.arange(1024 * 2048, device="cuda",
                                                       dtype=torch.int32).view(1024, 2048))).sum())
        print(json.dumps({"config": cfg, "t": t,
                          "bits_us_per_frame": round(e0.elapsed_time(e1) * 1e3 / n / B, 2),
                          "labels_us_per_frame": round(e1.elapsed_time(e2) * 1e3 / n / B, 2),
                          "components_frame0": comps}), flush=True)
