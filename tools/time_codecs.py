"""Time the device input codecs at C3 frame size
(2048x1024) with CUDA events; prints one JSON line per kernel with the
algorithmic bytes per pixel and the fraction of MEASURED_PEAKS.json's HBM
bandwidth.  Inputs are larger than L2 (>= 64 frames)."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2504_15121_b200 import KernelSpec, device, scenes  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
H, W = 1024, 2048
peaks = json.loads(Path("MEASURED_PEAKS.json").read_text()) if Path("MEASURED_PEAKS.json").exists() else {}
peak = float(peaks.get("hbm_gbs", 6542.1))
sc = scenes.street_scene(W, H)
clean = scenes.raycast(sc)[0]
rng = np.random.default_rng(0)
q = np.clip(np.rint((clean + rng.normal(0, 0.2, clean.shape)) * 256 + 1), 1, 65535)
q[~np.isfinite(clean)] = 0
raw = torch.from_numpy(q.astype(np.uint16)).cuda().expand(B, -1, -1).contiguous()


def timed(fn, n=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n  # ms per call


def report(name, ms, bpp, extra=None):
    us = ms * 1e3 / B
    gbs = bpp * B * H * W / (ms * 1e-3) / 1e9
    line = {"kernel": name, "us_per_frame": round(us, 2), "bytes_per_px": bpp,
            "achieved_gbps": round(gbs, 1), "peak_gbps": peak, "frac": round(gbs / peak, 3),
            "mpx_per_s": round(H * W / us, 1)}
    line.update(extra or {})
    print(json.dumps(line), flush=True)


o32 = torch.empty(B, H, W, device="cuda")
o64 = torch.empty(B, H, W, device="cuda", dtype=torch.float64)
report("dequant_png16->f32", timed(lambda: device.dequant_png16(raw, 256.0, 0, dtype=torch.float32, out=o32)), 6)
report("dequant_png16->f64", timed(lambda: device.dequant_png16(raw, 256.0, 0, out=o64)), 10)
payload = torch.empty(B * H * W * 4, dtype=torch.uint8, device="cuda")
payload.view(torch.float32).copy_(o32.reshape(-1))
for be in (False, True):
    report(f"decode_pfm(be={be})", timed(lambda: device.decode_pfm(payload, H, W, 1, be, out=o32)), 8)
out6 = torch.empty(B, H, W, 6, device="cuda")
mask = torch.empty(B, H, W, dtype=torch.uint8, device="cuda")
d = device.dequant_png16(raw, 256.0, 0, dtype=torch.float32)
k = KernelSpec.square(9)
report("fused_fp32_k9", timed(lambda: device.oriented_points(d, sc.rig, k, out=out6, mask=mask)), 29)
report("fused_png16_k9", timed(lambda: device.oriented_points_png16(raw, sc.rig, k, scale=256.0,
                                                                    out=out6, mask=mask)), 27)
