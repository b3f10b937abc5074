import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2504_15121_b200 import device, scenes
sc = scenes.street_scene(2048, 1024)
clean = torch.from_numpy(scenes.raycast(sc)[0].astype(np.float32)).cuda()
B = 64
d = clean.expand(B, -1, -1).contiguous() + 0.2 * torch.randn(B, 1024, 2048, device='cuda')
out = torch.empty(B, 1024, 2048, 6, device='cuda')
bits = torch.empty(B, 1024, 64, dtype=torch.int32, device='cuda')
bits2 = torch.empty_like(bits)
def t(fn, n=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n / B
print("fused only      ", round(t(lambda: device.oriented_points(d, sc.rig, 9, out=out)), 2))
print("fused + bits    ", round(t(lambda: device.oriented_points_bits(d, sc.rig, 9, 0.2, out=out, bits=bits)), 2))
print("standalone bits ", round(t(lambda: device.passable_bits(d, sc.rig, 0.2, bits=bits2)), 2))
device.oriented_points_bits(d, sc.rig, 9, 0.2, out=out, bits=bits)
device.passable_bits(d, sc.rig, 0.2, bits=bits2)
torch.cuda.synchronize()
print("bits equal", torch.equal(bits, bits2))
