"""Host cost of one call (launch overhead) vs device time, single C3 frame:
back-to-back launches between one pair of events (device-bound when the
host runs ahead) and the per-call host time of the Python and C-ABI paths."""
import ctypes
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_15121_b200 import KernelSpec, _native, device, scenes  # noqa: E402

sc = scenes.street_scene(2048, 1024)
d = torch.from_numpy(scenes.add_gaussian_noise(scenes.raycast(sc)[0], 0.2, 1).astype(np.float32)).cuda()[None]
out = torch.empty(1, 1024, 2048, 6, device="cuda")
labels = torch.empty(1, 1024, 2048, dtype=torch.int32, device="cuda")
ws = device.ccl_workspace(1, 1024, 2048, d.device)
res = {}
for name, fn in (("points", lambda: device.oriented_points(d, sc.rig, 9, out=out)),
                 ("pipeline", lambda: device.pipeline(d, sc.rig, 9, 0.2, out=out, labels=labels,
                                                      workspace=ws))):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50):
        fn()
    host = (time.perf_counter() - t0) / 50
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(50):
        fn()
    e1.record()
    torch.cuda.synchronize()
    res[name] = {"host_us_per_call": round(host * 1e6, 1),
                 "device_us_per_call_back_to_back": round(e0.elapsed_time(e1) * 1e3 / 50, 1)}
# the raw C ABI call (no Python-side argument building)
lib = _native.load()
plan = _native.plan(0)
rs = _native.rig_struct(sc.rig)
off = _native.offsets_array(KernelSpec.square(9).offsets)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    lib.sn_oriented_points(plan, d.data_ptr(), 1, 1024, 2048, ctypes.byref(rs), off.ctypes.data,
                           len(off), out.data_ptr(), None, st)
res["abi_points_host_us_per_call"] = round((time.perf_counter() - t0) / 50 * 1e6, 1)
torch.cuda.synchronize()
print(json.dumps(res))
