"""Per-phase clock64 cycles of the tile union-find (experiment build with
SN_CCL_PROF, exp/libsn_prof.so): cycles summed over CTAs (thread 0 of each)."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_15121_b200 import _native, device, scenes  # noqa: E402

lib = _native.load()
prof = getattr(lib, "sn_debug_ccl_prof")
buf = (ctypes.c_ulonglong * 16)()
B = 64
sc = scenes.street_scene(2048, 1024)
base = torch.from_numpy(scenes.raycast(sc)[0].astype(np.float32)).cuda()
d = base.expand(B, -1, -1).contiguous() + 0.2 * torch.randn(B, 1024, 2048, device="cuda")
ws = device.ccl_workspace(B, 1024, 2048, d.device)
lab = torch.empty(B, 1024, 2048, dtype=torch.int32, device="cuda")
for t in (0.05, 0.2, 1.0):
    bits = device.passable_bits(d, sc.rig, t)
    device.labels_from_bits(bits, 2048, out=lab, workspace=ws)
    torch.cuda.synchronize()
    prof(buf, 1)
    device.labels_from_bits(bits, 2048, out=lab, workspace=ws)
    torch.cuda.synchronize()
    prof(buf, 1)
    tiles = B * 128
    print(json.dumps({"t": t, "cycles_per_tile": [round(buf[i] / tiles) for i in range(5)],
                      "phases": ["A parents", "B jumping", "C unions", "D roots", "E labels"]}))
