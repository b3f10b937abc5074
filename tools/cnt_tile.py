"""Union-find operation counts per tile (experiment build with SN_CCL_CNT)."""
import ctypes
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_15121_b200 import _native, device, scenes  # noqa: E402

lib = _native.load()
cnt = getattr(lib, "sn_debug_ccl_cnt")
buf = (ctypes.c_ulonglong * 8)()
B = 16
sc = scenes.street_scene(2048, 1024)
base = torch.from_numpy(scenes.raycast(sc)[0].astype(np.float32)).cuda()
d = base.expand(B, -1, -1).contiguous() + 0.2 * torch.randn(B, 1024, 2048, device="cuda")
for t in (0.05, 0.2, 1.0):
    bits = device.passable_bits(d, sc.rig, t)
    torch.cuda.synchronize()
    cnt(buf, 1)
    device.labels_from_bits(bits, 2048)
    torch.cuda.synchronize()
    cnt(buf, 1)
    tiles = B * 128
    names = ["unite_calls", "find_steps", "unite_loops", "atomics", "root_walk_steps"]
    print(json.dumps({"t": t, **{n: round(buf[i] / tiles, 1) for i, n in enumerate(names)}}))
