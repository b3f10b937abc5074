"""Small end-to-end run of every kernel for compute-sanitizer (memcheck /
racecheck / synccheck): fused pass (fp32 / fp64 / generic), bits, labeller
(all modes), strips, cloud compaction, adaptive ST/CD."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2504_15121_b200 import KernelSpec, StarConfig, device, scenes
from paper_2504_15121_b200.parallel import StripPlan, local_strip_frame

sc = scenes.street_scene(300, 140)
d = scenes.add_gaussian_noise(scenes.raycast(sc)[0], 0.5, 1).astype(np.float32)
d[50:60, 100:120] = np.nan
dt = torch.from_numpy(np.stack([d, d[::-1].copy()])).cuda()
r = sc.rig
mask = torch.empty(dt.shape, dtype=torch.uint8, device="cuda")
pts = device.oriented_points(dt, r, 9, mask=mask)
device.oriented_points(dt.double(), r, 9)
device.oriented_points(dt, r, KernelSpec(np.array([[0, 0], [1, 0], [0, 1], [-1, -1]])))
device.affine(dt, 5)
p, bits = device.oriented_points_bits(dt, r, 9, 0.2)
device.labels_from_bits(bits, 300)
device.component_labels(dt, r, 0.2)
device.labels_from_passable(device.passable(dt, r, 0.2))
device.pipeline(dt, r, 9, 0.2)
local_strip_frame(dt[0].contiguous(), StripPlan.for_kernel(140, 300, 3, 9), r, 9, 0.2)
device.compact_cloud(pts, mask)
device.adaptive_points(dt, r, StarConfig(stop="cd", threshold=0.1))
device.adaptive_points(dt, r, StarConfig(stop="st", threshold=0.5, shared_range=True))
# widths TMA cannot address: pitched input (302), pitched input + output (301, 299)
for w in (302, 301, 299):
    dw = dt[:, :, :w].contiguous()
    device.oriented_points(dw, r, 9, mask=torch.empty(dw.shape, dtype=torch.uint8, device="cuda"))
    device.oriented_points(dw.double(), r, 5)
    device.pipeline(dw, r, 9, 0.2)
raw = torch.clamp(dt.nan_to_num(0.0) * 256 + 1, 0, 65535).to(torch.int32).to(torch.int16)
device.oriented_points_png16(raw, r, 9)
device.oriented_points_png16(raw[:, :, :301].contiguous(), r, 9)
torch.cuda.synchronize()
print("sanitize run ok")
