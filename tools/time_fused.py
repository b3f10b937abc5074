import sys, time, torch, numpy as np
sys.path.insert(0, '.')
from paper_2504_15121_b200 import device, scenes
sc = scenes.street_scene(2048, 1024)
clean = torch.from_numpy(scenes.raycast(sc)[0].astype(np.float32)).cuda()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
d = clean.expand(B, -1, -1).contiguous() + 0.2 * torch.randn(B, 1024, 2048, device='cuda')
out = torch.empty(B, 1024, 2048, 6, device='cuda')
for _ in range(3): device.oriented_points(d, sc.rig, 9, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
n = 20
for _ in range(n): device.oriented_points(d, sc.rig, 9, out=out)
e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / n / B
print(f"fused: {us:.2f} us/frame  {28*2048*1024/us/1e3:.0f} GB/s")
