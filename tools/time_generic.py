"""Generic (any offset pattern) pass vs the square fast path, C3 frames, CUDA
events: us/frame for the forced-generic 9x9 square and a few off-square
patterns (cross, sparse, 19x19 square)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_15121_b200 import KernelSpec, device, scenes  # noqa: E402

B = 16
sc = scenes.street_scene(2048, 1024)
base = torch.from_numpy(scenes.raycast(sc)[0].astype(np.float32)).cuda()
d = base.expand(B, -1, -1).contiguous() + 0.2 * torch.randn(B, 1024, 2048, device="cuda")
out = torch.empty(B, 1024, 2048, 6, device="cuda")


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) * 1e3 / reps / B, 2)


res = {"fast_9x9": timed(lambda: device.oriented_points(d, sc.rig, 9, out=out)),
       "generic_9x9": timed(lambda: device.oriented_points(d, sc.rig, 9, out=out, generic=True)),
       "cross4": timed(lambda: device.oriented_points(
           d, sc.rig, KernelSpec(np.array([[1, 0], [-1, 0], [0, 1], [0, -1]])), out=out)),
       "sparse6": timed(lambda: device.oriented_points(
           d, sc.rig, KernelSpec(np.array([[0, 0], [2, 1], [1, 2], [-2, -1], [3, -2], [-1, 3]])),
           out=out)),
       "square_19x19": timed(lambda: device.oriented_points(d, sc.rig, 19, out=out), reps=1),
       "affine_9x9_fp64_out": timed(lambda: device.affine(d, 9))}
print(json.dumps({"us_per_frame": res}))
