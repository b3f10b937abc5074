"""Probe: do the passable-bits kernel (ALU-bound) and the labeller (latency-
bound) overlap when run concurrently on two streams?  Prints sequential vs
concurrent time per frame.  Not part of the product."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2504_15121_b200 import device, scenes

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
sc = scenes.street_scene(2048, 1024)
clean = torch.from_numpy(scenes.raycast(sc)[0].astype(np.float32)).cuda()
d = clean.expand(2 * B, -1, -1).contiguous() + 0.2 * torch.randn(2 * B, 1024, 2048, device="cuda")
bits = device.passable_bits(d, sc.rig, 0.2)
lab = torch.empty(2 * B, 1024, 2048, dtype=torch.int32, device="cuda")
ws = device.ccl_workspace(B, 1024, 2048, d.device)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def seq():
    device.passable_bits(d[:B], sc.rig, 0.2, bits=bits[:B])
    device.labels_from_bits(bits[B:], 2048, out=lab[B:], workspace=ws)


def conc():
    with torch.cuda.stream(s1):
        device.passable_bits(d[:B], sc.rig, 0.2, bits=bits[:B])
    with torch.cuda.stream(s2):
        device.labels_from_bits(bits[B:], 2048, out=lab[B:], workspace=ws)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


for name, fn in [("sequential", seq), ("concurrent", conc), ("sequential", seq), ("concurrent", conc)]:
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    s1.wait_stream(torch.cuda.current_stream())
    s2.wait_stream(torch.cuda.current_stream())
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) * 1e3 / 10 / B:.2f} us/frame")
