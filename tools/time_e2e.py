"""End-to-end host-buffer pipeline (sn_pipeline_host: pinned host in/out, H2D +
compute + D2H) at C3, 64-frame steps, wall time per step; the pinned-copy
peaks of the same process for the bound."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2504_15121_b200 as sn  # noqa: E402
from paper_2504_15121_b200 import _native, scenes  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
H, W = 1024, 2048
sc = scenes.street_scene(W, H)
base = torch.from_numpy(scenes.raycast(sc)[0].astype(np.float32))
host_in = (base.expand(B, -1, -1) + 0.2 * torch.randn(B, H, W)).contiguous().pin_memory()
host_out = torch.empty((B, H, W, 6), dtype=torch.float32).pin_memory()
host_lab = torch.empty((B, H, W), dtype=torch.int32).pin_memory()
lib = _native.load()
plan = _native.plan(0)
rs = _native.rig_struct(sc.rig)
off = _native.offsets_array(sn.KernelSpec.square(9).offsets)


def step():
    rc = lib.sn_pipeline_host(plan, host_in.data_ptr(), B, H, W, ctypes.byref(rs), off.ctypes.data,
                              len(off), 0.2, host_out.data_ptr(), None, host_lab.data_ptr())
    _native.check(rc, "host pipeline")


step()
best = 1e9
for _ in range(4):
    t0 = time.perf_counter()
    step()
    best = min(best, time.perf_counter() - t0)
d2h = B * H * W * 28
dev = torch.empty(d2h // 4, dtype=torch.float32, device="cuda")
hb = torch.empty(d2h // 4, dtype=torch.float32).pin_memory()
torch.cuda.synchronize()
t0 = time.perf_counter()
hb.copy_(dev, non_blocking=True)
torch.cuda.synchronize()
d2h_s = time.perf_counter() - t0
print(f"e2e {best * 1e3:.2f} ms/step  {B * H * W / best / 1e6:.0f} Mpx/s  "
      f"(one D2H of the step's bytes: {d2h_s * 1e3:.2f} ms = {d2h / d2h_s / 1e9:.1f} GB/s; "
      f"frac {d2h_s / best:.3f})")
