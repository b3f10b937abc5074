import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from conftest import _load
from helpers import rig_of
from paper_2504_15121_b200 import device, KernelSpec
cases = _load("fixed_cases.npz")
for name in sys.argv[1:]:
    c = cases[name]
    d = torch.from_numpy(c["d"]).cuda().float()
    for generic in (False, True):
        m = torch.zeros(d.shape, dtype=torch.uint8, device='cuda')
        out = device.oriented_points(d, rig_of(c["rig"]), KernelSpec(c["offsets"]), mask=m, generic=generic)
        torch.cuda.synchronize()
        mm = m.cpu().numpy().astype(bool); o = out[0].cpu().numpy()
        print(name, "generic" if generic else "fast", d.shape, "mask eq", np.array_equal(mm, c["nmask"]), "got", mm.sum(), "want", c["nmask"].sum())
        if not np.array_equal(mm, c["nmask"]):
            print(mm.astype(int)[:6, :16]); print(c["nmask"].astype(int)[:6, :16])
            print(o[2, 2], c["normals"][2, 2], c["points"][2,2])
