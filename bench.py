#!/usr/bin/env python
"""Benchmark of the B200 hot path (BASELINE.json metric).

Headline workload (N=1, and per rank for N>1): configuration C3 -- synthetic
2048x1024 street-scene disparities, 256 frames per GPU (weak scaling: each
rank owns its own 256-frame shard, no data-path collective).  One step = the
full north-star pipeline over the batch: fused fixed-kernel pass (k = 9 LSQ
fit + closed-form normal + triangulation -> dense [B,H,W,6] fp32 oriented
points), the ST-passable bit mask (t = 0.2) and the 8-connected component
labels from it.  Inputs are resident in HBM; 2.1 GB in / 12.9 GB out per
step, far larger than the 126 MB L2, so no flush is needed between steps.

Reported: value = whole-job Mpx/s (all ranks) from CUDA events on the launch
stream, max over ranks; roofline of the dominant kernel (the fused pass) from
its own CUDA-event time inside the timed region; e2e through the C-ABI
host-buffer entry (pinned host in/out, copies inside the timed region) with
its own PCIe roofline; cpu_baseline = the reference package itself
(baseline/_ref, installed by tools/install_reference.sh) on a bounded sample,
else the oracle port.  After the headline, the other named configs are
measured briefly (`configs`): C2 (2888x1920 sphere, L2 flushed between
repetitions), C4 (64 noisy frames with holes at t = 0.05 / 0.2 / 1.0) and C5
(7680x4320 in one strip per rank: halo exchange, strip pass, NCCL seam
all-gather and relabel inside the timed region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

With --gpus N > 1 and no torchrun environment the script re-launches itself
under torch.distributed.run with N ranks (one per GPU).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import shutil
import socket
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
REF_PATH = ROOT / "baseline" / "_ref"

METRIC = "megapixels/sec (oriented points) at 2048×1024, 1/2/4/8 B200; % HBM roofline"
H, W, FRAMES, KSIZE, T_ST = 1024, 2048, 256, 9, 0.2
BYTES_PER_PX = 28  # algorithmic: 4 B fp32 disparity in + 24 B (x,y,z,nx,ny,nz) out
WORKLOAD = "C3 2048x1024 street, fixed 9x9 pass + ST(t=0.2) component labels"
IO = "fp32 disparity in, fp32 AoS-6 record out; exact fp64 sums, fp32 epilogue"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=60)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--frames", type=int, default=FRAMES, help="frames per GPU")
    ap.add_argument("--pipeline", choices=["full", "points"], default="full")
    ap.add_argument("--e2e-steps", type=int, default=7)
    ap.add_argument("--e2e-frames", type=int, default=64,
                    help="frames per rank in the e2e leg (pinned host buffers ~70 MB/frame)")
    ap.add_argument("--cpu-frames", type=int, default=16, help="cpu_baseline sample (frames)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the C2/C4/C5 legs")
    ap.add_argument("--extras", action="store_true",
                    help="also time the next-row kernels (adaptive, cloud, evaluation, PNG16 "
                         "input) briefly after the headline measurement")
    ap.add_argument("--no-extras", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--dry-run", action="store_true",
                    help="rank plumbing only (gloo on CPU, no GPU work): prints the ranks seen")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def relaunch_under_torchrun(args) -> int:
    """--gpus N > 1 without a torchrun environment: start N ranks on this node
    (the driver's own launch line, 127.0.0.1 rendezvous)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd)


def cpu_model() -> str:
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def street_clean():
    from paper_2504_15121_b200 import scenes
    sc = scenes.street_scene(W, H)
    disp, _, _ = scenes.raycast(sc)
    return sc.rig, disp


# ---------------------------------------------------------------------------
# CPU legs: the reference package itself (baseline/_ref) when installed, else
# the oracle port of its algorithm -- bench-only use


def reference_step_fn(rig, threads):
    """(kind, fn(d) -> None) running the reference's hot path on one float64
    frame: estimate_normals_fixed through its own bench closure
    (bench.py:61-73 make_bench_callable 'affine-fixed', prebuilt kernels),
    triangulate_grid, and the ST passable set depth_laplacian(depth_field)
    <= t labelled 8-connected (scipy.ndimage.label + min-index relabel, as the
    oracle: the reference has no labeller)."""
    from oracle import stereonorm_oracle as orc
    if (REF_PATH / "stereonorm").exists():
        sys.path.insert(0, str(REF_PATH))
        try:
            import stereonorm as sn
        finally:
            sys.path.remove(str(REF_PATH))
        rrig = sn.StereoRig(rig.fx, rig.fy, rig.u0, rig.v0, rig.baseline)

        def fn(d):
            field = sn.ScalarField.from_array(d)
            sn.bench.make_bench_callable("affine-fixed", field, rrig, KSIZE, threads=threads)()
            sn.triangulate_grid(field, rrig)
            e = sn.depth_laplacian(sn.depth_field(field, rrig))
            with np.errstate(invalid="ignore"):
                orc.label_components(e.mask & (e.values <= T_ST))
        return "reference", fn
    orig = orc.Rig(rig.fx, rig.fy, rig.u0, rig.v0, rig.baseline)

    def fn(d):
        orc.oriented_points(d, orig, KSIZE, threads=threads)
        orc.ccl_labels(d, orig, T_ST)
    return "port", fn


def cpu_sample(rig, clean, n_frames, threads):
    """Time the reference algorithm over n_frames C3 frames with the
    reference's own method (bench.py:38-52: 1 warm-up, perf_counter)."""
    from paper_2504_15121_b200 import scenes
    kind, fn = reference_step_fn(rig, threads)
    frames = [scenes.add_gaussian_noise(clean, 0.2, i).astype(np.float32).astype(np.float64)
              for i in range(n_frames + 1)]
    fn(frames[0])  # warm-up
    t0 = time.perf_counter()
    for d in frames[1:]:
        fn(d)
    dt = time.perf_counter() - t0
    return kind, n_frames * H * W / 1e6 / dt, dt


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    rig, clean = street_clean()
    threads = os.cpu_count() or 1
    per_step = 2  # bounded sample per step (frames)
    from paper_2504_15121_b200 import scenes
    kind, fn = reference_step_fn(rig, threads)
    frames = [scenes.add_gaussian_noise(clean, 0.2, i).astype(np.float32).astype(np.float64)
              for i in range(per_step)]

    def step():
        for d in frames:
            fn(d)

    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    sec = sum(times) / len(times)
    val = per_step * H * W / 1e6 / sec
    what = ("the reference package (baseline/_ref stereonorm 0.1.0): estimate_normals_fixed "
            "via its bench closure + triangulate_grid + depth_laplacian(depth_field) <= t, "
            "scipy 8-connected labels" if kind == "reference" else
            "oracle port of estimate_normals_fixed + triangulate_grid + ST labels")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "Mpx/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (C3 street scene, PCG64 noise sigma 0.2, fp32-representable values)",
        "config": {"workload": WORKLOAD, "height": H, "width": W, "kernel": KSIZE},
        "cpu_baseline": {"value": val, "unit": "Mpx/s", "cores": threads, "kind": kind,
                         "cpu_model": cpu_model(),
                         "sample": f"{per_step} C3 frames/step x {args.steps} steps, {what}, "
                                   f"threads={threads}"},
        "e2e": {"value": val, "unit": "Mpx/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# clocks during the timed region


class ClockSampler:
    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        if not shutil.which("nvidia-smi"):
            return
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        self.proc = subprocess.Popen(
            ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}", "--format=csv,noheader,nounits",
             "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.th.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# GPU arm


def measured_hbm_peak() -> float:
    """HBM GB/s: MEASURED_PEAKS.json (driver-written copy bandwidth), else the
    profiling recipe's fallback."""
    pk = ROOT / "MEASURED_PEAKS.json"
    peaks = json.loads(pk.read_text()) if pk.exists() else {}
    return float(peaks.get("hbm_gbs", 6650.0))


def pcie_peaks(dev, nbytes=1 << 30):
    """Pinned host<->device copy bandwidth (GB/s) per direction: 1 GB as one
    cudaMemcpyAsync or as two halves on two streams, best of 6, host wall
    clock around a synchronised copy -- the ceiling of the e2e leg."""
    import torch
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    res = {}
    s_a, s_b = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    half = nbytes // 2
    for name, (dst, src) in (("h2d_gbs", (d, h)), ("d2h_gbs", (h, d))):
        best = 0.0
        for rep in range(6):
            # one copy, or the two halves on two streams (the e2e pipeline keeps
            # several copies queued): the best of either is the ceiling
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            if rep % 2 == 0:
                dst.copy_(src, non_blocking=True)
            else:
                with torch.cuda.stream(s_a):
                    dst[:half].copy_(src[:half], non_blocking=True)
                with torch.cuda.stream(s_b):
                    dst[half:].copy_(src[half:], non_blocking=True)
            torch.cuda.synchronize()
            best = max(best, nbytes / (time.perf_counter() - t0) / 1e9)
        res[name] = round(best, 2)
    # both directions at once (the e2e leg overlaps them on two streams)
    h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d2 = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    res["duplex_gbs"] = round(2 * nbytes / (time.perf_counter() - t0) / 1e9, 2)
    del h, d, h2, d2
    return res


def copy_schedule_ms(dev, B, H, W, full):
    """The host pipeline's copies alone: sn_pipeline_host's chunks (1, 2, 4, ..
    frames up to ~16 Mpx, sn_api.cu host_pipeline) and its event graph over
    three streams (H2D of chunk c after chunk c-2's "compute", "compute" after
    its H2D and chunk c-2's D2H, D2H after the "compute"), with no kernels: what
    the PCIe link alone allows in that schedule (both directions share the
    full-duplex link).  Best of 3, wall clock around synchronised steps."""
    import torch
    px = H * W
    chunk = min(B, max(1, (16 << 20) // px))
    sizes, f = [], 0
    while f < B:
        n = min(B - f, chunk if (1 << len(sizes)) >= chunk else 1 << len(sizes))
        sizes.append(n)
        f += n
    n_in, n_out = chunk * px * 4, chunk * px * (28 if full else 24)
    h_in = torch.empty(B * px * 4, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(B * px * (28 if full else 24), dtype=torch.uint8).pin_memory()
    d_in = [torch.empty(n_in, dtype=torch.uint8, device=dev) for _ in range(2)]
    d_out = [torch.empty(n_out, dtype=torch.uint8, device=dev) for _ in range(2)]
    s_h, s_c, s_d = (torch.cuda.Stream(dev) for _ in range(3))
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]

    def step():
        f0 = 0
        for c, n in enumerate(sizes):
            k = c & 1
            if c >= 2:
                s_h.wait_event(ev_done[k])
                s_c.wait_event(ev_out[k])
            bi, bo = n * px * 4, n * px * (28 if full else 24)
            with torch.cuda.stream(s_h):
                d_in[k][:bi].copy_(h_in[f0 * px * 4:f0 * px * 4 + bi], non_blocking=True)
            ev_in[k].record(s_h)
            s_c.wait_event(ev_in[k])
            ev_done[k].record(s_c)
            s_d.wait_event(ev_done[k])
            o = f0 * px * (28 if full else 24)
            with torch.cuda.stream(s_d):
                if full:  # records, then labels: two copies as in the pipeline
                    r = n * px * 24
                    h_out[o:o + r].copy_(d_out[k][:r], non_blocking=True)
                    h_out[o + r:o + bo].copy_(d_out[k][r:bo], non_blocking=True)
                else:
                    h_out[o:o + bo].copy_(d_out[k][:bo], non_blocking=True)
            ev_out[k].record(s_d)
            f0 += n

    best = 1e9
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        step()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    del h_in, h_out, d_in, d_out
    return best * 1e3


def flush_l2(buf, sink):
    # read 256 MB (clean lines: evicts the 126 MB L2 without leaving dirty
    # lines for the timed kernel to write back)
    torch_sum = buf.sum(dtype=None)
    sink.copy_(torch_sum)


def next_row_timings(dN, outN, rig, dev):
    """us/frame of the f1-f4 kernels (CUDA events, 3 reps after one untimed
    call): the adaptive walks on 8 C3 frames, the streaming rows (PNG16 fused
    pass, cloud compaction, evaluation) on all of dN (64 frames: whole waves)."""
    import torch
    from paper_2504_15121_b200 import StarConfig, device, scenes
    n = dN.shape[0]
    d8, out8 = dN[:8], outN[:8]
    mask = torch.empty(dN.shape, dtype=torch.uint8, device=dev)
    sc = scenes.street_scene(W, H)
    gt = torch.from_numpy(np.ascontiguousarray(scenes.raycast(sc)[2])).to(dev)
    gt = gt.expand(n, -1, -1, -1).contiguous()
    gm = torch.isfinite(gt).all(-1).to(torch.uint8)
    raw = torch.clamp(torch.round(dN * 256 + 1), 1, 65535).to(torch.int32).to(torch.uint16)
    cd, st = StarConfig(stop="cd", threshold=0.1), StarConfig(stop="st", threshold=0.2)

    def timed(fn, frames, reps=3):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return round(e0.elapsed_time(e1) * 1e3 / reps / frames, 2)

    gpu = {
        "frames_adaptive": 8,
        "frames_streaming": n,
        "adaptive_cd_s10_d8": timed(lambda: device.adaptive_points(d8, rig, cd, out=out8), 8),
        "adaptive_st_s10_d8": timed(lambda: device.adaptive_points(d8, rig, st, out=out8), 8),
        "fused_pass_png16_input": timed(lambda: device.oriented_points_png16(
            raw, rig, KSIZE, scale=256.0, out=outN), n),
        "fused_pass_fp64_input": timed(lambda: device.oriented_points(
            dN.double(), rig, KSIZE, out=outN), n),
    }
    # the fixed-pass records + mask the cloud and the evaluation consume
    device.oriented_points(dN, rig, KSIZE, out=outN, mask=mask)
    gpu["compact_cloud"] = timed(lambda: device.compact_cloud(outN, mask), n)
    gpu["angular_error_and_stats"] = timed(lambda: device.angular_error(outN, gt, gm), n)
    # HBM rows: algorithmic bytes per frame / time vs the measured copy peak
    keep = float(mask.float().mean())
    peak = measured_hbm_peak()
    roof = {}
    for name, bpp in (("fused_pass_png16_input", 2 + 24), ("compact_cloud", 1 + 48 * keep)):
        gbs = bpp * H * W / (gpu[name] * 1e-6) / 1e9
        roof[name] = {"bytes_per_px": round(bpp, 3), "achieved_gbs": round(gbs, 1),
                      "frac": round(gbs / peak, 4) if peak else None}
    return gpu, roof, (dN[0].double().cpu().numpy(), gt[0].cpu().numpy(), gm[0].cpu().numpy())


def next_row_cpu(d, gt_n, gt_m, rig):
    """us/frame of the reference algorithms of the f1-f4 rows (the oracle port,
    one C3 frame, numpy on the host; bench-only use of oracle/)."""
    from oracle import stereonorm_oracle as orc
    orig = orc.Rig(rig.fx, rig.fy, rig.u0, rig.v0, rig.baseline)

    def t(fn):
        t0 = time.perf_counter()
        r = fn()
        return round((time.perf_counter() - t0) * 1e6, 1), r

    res = {"frames": 1, "cores": 1}
    res["adaptive_cd_s10_d8"], _ = t(lambda: orc.estimate_normals_adaptive(
        d, orig, orc.Star(stop="cd", threshold=0.1)))
    res["adaptive_st_s10_d8"], _ = t(lambda: orc.estimate_normals_adaptive(
        d, orig, orc.Star(stop="st", threshold=0.2)))
    raw = np.clip(np.round(d * 256 + 1), 1, 65535).astype(np.int64)

    def png_fused():
        v, _ = orc.dequant_png16(raw, 256.0, 0)
        return orc.oriented_points(v, orig, KSIZE, threads=1)

    res["fused_pass_png16_input"], (p6, ok) = t(png_fused)
    res["compact_cloud"], _ = t(lambda: orc.ply_keep(p6, ok))
    res["angular_error_and_stats"], _ = t(
        lambda: orc.summarize(*orc.angular_error_map(p6[..., 3:], ok, gt_n, gt_m)))
    return res


def other_configs(dev, rank, world, disp_buf, out_buf, lab_buf, ws, bits_buf):
    """C2 / C4 / C5 (BASELINE.json configs 1, 3, 4), CUDA events on the launch
    stream, a few repetitions each after one untimed call.  C4 reuses the C3
    buffers (same frame shape); C2 flushes L2 between repetitions (its 155 MB
    step is about the L2 size); C5 runs one strip per rank (world strips)."""
    import torch
    import torch.distributed as dist
    from scipy import ndimage
    from paper_2504_15121_b200 import device, scenes
    from paper_2504_15121_b200.parallel import StripPlan, distributed_strip_frame, \
        local_strip_frame
    stream = torch.cuda.current_stream(dev)
    res = {}

    def ev_time(fn, reps, flush=None):
        # every repetition (flush, events, launches) is enqueued before one
        # synchronisation: the host runs ahead, so the events bracket device
        # time only, not the host's per-call launch cost
        evs = []
        for _ in range(reps):
            if flush is not None:
                flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in evs) / reps

    # C2: 2888x1920 sphere, one frame, full pipeline; L2 flushed before each rep
    sp = scenes.sphere_scene(2888, 1920)
    d2 = torch.from_numpy(scenes.add_gaussian_noise(scenes.raycast(sp)[0], 0.2, 7)
                          .astype(np.float32)).to(dev)[None]
    o2 = torch.empty((1, 1920, 2888, 6), dtype=torch.float32, device=dev)
    l2 = torch.empty((1, 1920, 2888), dtype=torch.int32, device=dev)
    ws2 = device.ccl_workspace(1, 1920, 2888, dev)
    scratch = torch.ones(64 << 20, dtype=torch.float32, device=dev)
    sink = torch.empty((), dtype=torch.float32, device=dev)
    fn2 = lambda: device.pipeline(d2, sp.rig, KSIZE, T_ST, out=o2, labels=l2, workspace=ws2)  # noqa
    fn2()
    ms2 = ev_time(fn2, 10, lambda: flush_l2(scratch, sink))
    ms2p = ev_time(lambda: device.oriented_points(d2, sp.rig, KSIZE, out=o2), 10,
                   lambda: flush_l2(scratch, sink))
    px2 = 2888 * 1920
    res["C2"] = {"workload": "2888x1920 sphere (sigma 0.2), 1 frame, fixed 9x9 + ST(0.2) labels",
                 "ms_per_frame": ms2, "value_mpx_s": px2 / 1e3 / ms2,
                 "fused_pass_ms": ms2p,
                 "fused_pass_frac_hbm": BYTES_PER_PX * px2 / (ms2p * 1e-3) / 1e9 /
                 measured_hbm_peak(),
                 "l2": "flushed (256 MB read) before each of 10 repetitions"}
    del d2, o2, l2, ws2

    # C4: 64 frames, sigma 1.0 + dilated holes, t = 0.05/0.2/1.0
    sc = scenes.street_scene(W, H)
    clean = scenes.raycast(sc)[0]
    n4 = min(64, disp_buf.shape[0])
    d4 = disp_buf[:n4]
    for i in range(n4):
        d = scenes.add_gaussian_noise(clean, 1.0, 4000 + i)
        holes = ndimage.binary_dilation(np.random.default_rng(1000 + i).random(d.shape) < 0.002,
                                        iterations=3)
        d4[i] = torch.from_numpy(np.where(holes, np.nan, d).astype(np.float32)).to(dev)
    c4 = {"workload": f"C4 2048x1024 street sigma 1.0 + 4.9% dilated holes, {n4} frames"}
    for t in (0.05, 0.2, 1.0):
        fb = lambda: device.passable_bits(d4, sc.rig, t, bits=bits_buf[:n4])  # noqa: E731
        fl = lambda: device.labels_from_bits(bits_buf[:n4], W, out=lab_buf[:n4],  # noqa: E731
                                             workspace=ws)
        fb(), fl()
        ms_b = ev_time(fb, 3)
        ms_l = ev_time(fl, 3)
        ncomp = int(torch.unique(lab_buf[0]).numel() - 1)
        c4[f"t={t}"] = {"bits_us_per_frame": ms_b * 1e3 / n4, "ccl_us_per_frame": ms_l * 1e3 / n4,
                        "components_frame0": ncomp}
    fp = lambda: device.pipeline(d4, sc.rig, KSIZE, T_ST, out=out_buf[:n4],  # noqa: E731
                                 labels=lab_buf[:n4], workspace=ws)
    fp()
    ms4 = ev_time(fp, 3)
    c4["pipeline_t0.2_us_per_frame"] = ms4 * 1e3 / n4
    c4["value_mpx_s"] = n4 * H * W / 1e3 / ms4
    res["C4"] = c4

    # C5: 7680x4320, one strip per rank (world strips): halo exchange, strip
    # pass, seam all-gather + relabel -- all inside the timed region
    sc5 = scenes.street_scene(7680, 4320)
    H5, W5 = 4320, 7680
    plan = StripPlan.for_kernel(H5, W5, world, KSIZE)
    r0, r1 = plan.owned(rank)
    full = scenes.add_gaussian_noise(scenes.raycast(sc5)[0], 0.2, 0).astype(np.float32)
    owned = torch.from_numpy(full[r0:r1]).to(dev)
    if world > 1:
        run5 = lambda: distributed_strip_frame(owned, plan, sc5.rig, KSIZE, T_ST)  # noqa: E731
    else:
        # one GPU holds the whole frame: one pipeline call; the 8-strip path
        # (block slicing, per-strip passes, host seam merge, relabel) is timed
        # beside it as the single-GPU stand-in of the multi-GPU partition
        dfull = torch.from_numpy(full).to(dev)[None]
        o5 = torch.empty((1, H5, W5, 6), dtype=torch.float32, device=dev)
        l5 = torch.empty((1, H5, W5), dtype=torch.int32, device=dev)
        ws5 = device.ccl_workspace(1, H5, W5, dev)
        run5 = lambda: device.pipeline(dfull, sc5.rig, KSIZE, T_ST, out=o5, labels=l5,  # noqa
                                       workspace=ws5)
        strips8 = lambda: local_strip_frame(dfull[0], StripPlan.for_kernel(H5, W5, 8, KSIZE),  # noqa
                                            sc5.rig, KSIZE, T_ST)
        strips8()
        ms_strips = ev_time(strips8, 3)
    run5()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms5 = ev_time(run5, 3)
    if world > 1:
        t5 = torch.tensor([ms5], dtype=torch.float64, device=dev)
        dist.all_reduce(t5, op=dist.ReduceOp.MAX)
        ms5 = float(t5.item())
    c5 = {"workload": "7680x4320 street (sigma 0.2), 1 frame, fixed 9x9 + ST(0.2) labels, " +
                      (f"{world} strips, one per rank: NCCL halo P2P, strip pass, seam "
                       "all-gather + relabel inside the timed region" if world > 1 else
                       "whole frame on 1 GPU"),
          "ms_per_frame": ms5, "value_mpx_s": H5 * W5 / 1e3 / ms5, "ranks": world}
    if world == 1:
        c5["strips8_sequential_ms_per_frame"] = ms_strips
    res["C5"] = c5
    return res


def dry_run(args):
    """Rank plumbing without a GPU: gloo all-reduce of ones over the ranks."""
    import torch
    import torch.distributed as dist
    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    t = torch.ones(1)
    if world > 1:
        dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks_seen": int(t.item()),
                          "gpus_arg": args.gpus}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch_under_torchrun(args))
    rank, world, local = dist_env()
    if world != args.gpus:
        if rank == 0:
            print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.dry_run:
        dry_run(args)
        return
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist
    from paper_2504_15121_b200 import _native, device

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    rig, clean = street_clean()
    B = args.frames
    # synthetic batch: the clean street disparity + per-frame N(0, 0.2) noise
    # (device RNG seeded by rank), fp32, resident in HBM
    g = torch.Generator(device=dev)
    g.manual_seed(1234 + rank)
    base = torch.from_numpy(clean.astype(np.float32)).to(dev)
    disp = torch.empty((B, H, W), dtype=torch.float32, device=dev)
    for i in range(B):
        disp[i] = base + 0.2 * torch.randn((H, W), generator=g, device=dev)
    out = torch.empty((B, H, W, 6), dtype=torch.float32, device=dev)
    labels = torch.empty((B, H, W), dtype=torch.int32, device=dev)
    ccl_ws = device.ccl_workspace(B, H, W, dev)
    stream = torch.cuda.current_stream(dev)

    bits = torch.empty((B, H, device.bit_words(W)), dtype=torch.int32, device=dev)

    def step(ev=None):
        # the fused pass, then the labels from the disparities (predicate bit
        # mask + labeller; from 128 frames on the library runs the two half
        # batches on two streams, joined back into this one) -- split so the
        # fused kernel's own time is bracketed by events on the launch stream
        if ev is not None:
            ev[0].record(stream)
        device.oriented_points(disp, rig, KSIZE, out=out)
        if ev is not None:
            ev[1].record(stream)
            ev[2].record(stream)
        if args.pipeline == "full":
            device.component_labels(disp, rig, T_ST, out=labels, workspace=ccl_ws)
        if ev is not None:
            ev[3].record(stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.2)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_start.record(stream)
    for k in range(args.steps):
        step(evs[k])
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = sampler.stop()

    total_ms = t_start.elapsed_time(t_end)
    fused_ms = [e[0].elapsed_time(e[1]) for e in evs]
    bits_ms = [e[1].elapsed_time(e[2]) for e in evs]
    ccl_ms = [e[2].elapsed_time(e[3]) for e in evs]
    stats = torch.tensor([total_ms, statistics.mean(fused_ms), statistics.mean(bits_ms),
                          statistics.mean(ccl_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.MAX)
    total_ms, fused_avg, bits_avg, ccl_avg = stats.tolist()
    ms_per_step = total_ms / args.steps
    px_step = B * H * W
    value = world * px_step / 1e6 / (ms_per_step / 1e3)

    # roofline of the dominant kernel (fused pass): algorithmic bytes / its event time
    pk = ROOT / "MEASURED_PEAKS.json"
    peak = measured_hbm_peak()
    fused_bytes = BYTES_PER_PX
    achieved = fused_bytes * px_step / (fused_avg / 1e3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / "ncu_summary.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get("fused_pass", {}).get("dram_bytes_per_launch_at_c3")

    # e2e through the C-ABI host-buffer entry (pinned host buffers): the same
    # pipeline (points + passable bits + labels) with H2D of the disparities
    # and D2H of the points and labels inside the timed region
    e2e = None
    if not args.no_e2e:
        Be = max(1, min(B, args.e2e_frames))
        host_in = disp[:Be].cpu().pin_memory()
        host_out = torch.empty((Be, H, W, 6), dtype=torch.float32).pin_memory()
        host_lab = torch.empty((Be, H, W), dtype=torch.int32).pin_memory()
        lib = _native.load()
        plan = _native.plan(local)
        rs = _native.rig_struct(rig)
        off = _native.offsets_array(__import__("paper_2504_15121_b200").KernelSpec.square(KSIZE).offsets)
        full = args.pipeline == "full"

        def host_step():
            if full:
                rc = lib.sn_pipeline_host(plan, host_in.data_ptr(), Be, H, W, ctypes.byref(rs),
                                          off.ctypes.data, len(off), T_ST, host_out.data_ptr(),
                                          None, host_lab.data_ptr())
            else:
                rc = lib.sn_oriented_points_host(plan, host_in.data_ptr(), Be, H, W, ctypes.byref(rs),
                                                 off.ctypes.data, len(off), host_out.data_ptr(),
                                                 None)
            _native.check(rc, "host pipeline")
            # the step's result is in host memory: read one value of each output
            return float(host_out[0, H // 2, W // 2, 5]) + (int(host_lab[0, H // 2, W // 2]) if full else 0)

        host_step()
        if world > 1:
            dist.barrier()
        # each step timed on the host clock around the blocking call; the
        # median step (the shared host's PCIe rate drifts from run to run)
        step_s = []
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            host_step()
            step_s.append(time.perf_counter() - t0)
        e2e_s = torch.tensor([statistics.median(step_s)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
        sec = float(e2e_s.item())
        px_e2e = Be * H * W
        h2d_b = int(px_e2e * 4)
        d2h_b = int(px_e2e * (24 + (4 if full else 0)))
        # the copy peaks vary from run to run on a shared host: measured twice
        # (after the e2e steps and once more), the better of each direction
        pa, pb = pcie_peaks(dev), pcie_peaks(dev)
        pcie = {k: max(pa[k], pb[k]) for k in pa}
        # PCIe bound of one step: both directions run concurrently on the
        # plan's copy streams, so the slower direction bounds the step
        bound_s = max(h2d_b / (pcie["h2d_gbs"] * 1e9), d2h_b / (pcie["d2h_gbs"] * 1e9))
        # the same chunks' copies with no compute (the duplex link gives a
        # concurrent D2H less than its solo peak): what the schedule allows
        copies_ms = copy_schedule_ms(dev, Be, H, W, full)
        e2e = {"value": world * px_e2e / 1e6 / sec, "unit": "Mpx/s",
               "frames_per_step_per_rank": Be,
               "frames_per_sec_per_gpu": Be / sec,
               "h2d_bytes_per_step": h2d_b,
               "d2h_bytes_per_step": d2h_b,
               "ms_per_step": sec * 1e3,
               "ms_per_step_each": [round(x * 1e3, 2) for x in step_s],
               "statistic": f"median of {args.e2e_steps} steps",
               "pcie_gbs": pcie,
               "bound_ms_per_step": bound_s * 1e3,
               "frac": bound_s / sec,
               "copies_only_ms_per_step": copies_ms,
               "frac_vs_copies_only": copies_ms / (sec * 1e3),
               "bound": "pcie (max of H2D bytes / pinned H2D peak, D2H bytes / pinned D2H peak)",
               "path": ("sn_pipeline_host" if full else "sn_oriented_points_host") +
                       " (pinned host in/out, 3-stream H2D/compute/D2H overlap)"}
        del host_in, host_out, host_lab

    # next rows of the scope table, timed briefly on 8 of the
    # same frames after the headline measurement: evidence, not the metric
    extras = extras_roof = extras_cpu = None
    if rank == 0 and world == 1 and args.extras and not args.no_extras:
        try:
            extras, extras_roof, host = next_row_timings(disp[:64], out[:64], rig, dev)
            if not args.no_cpu:
                extras_cpu = next_row_cpu(*host, rig)
        except Exception as exc:  # never let an extra cost the headline line
            extras = {"error": f"{type(exc).__name__}: {exc}"}

    configs = None
    if not args.no_configs:
        try:
            configs = other_configs(dev, rank, world, disp, out, labels, ccl_ws, bits)
        except Exception as exc:  # never let a side leg cost the headline line
            configs = {"error": f"{type(exc).__name__}: {exc}"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        kind, val, dt = cpu_sample(rig, clean, args.cpu_frames, threads)
        _, val1, dt1 = cpu_sample(rig, clean, 2, 1)
        cpu = {"value": val, "unit": "Mpx/s", "cores": threads, "kind": kind,
               "cpu_model": cpu_model(),
               "value_threads1": val1,
               "sample": f"{args.cpu_frames} C3 frames ({dt:.1f} s wall) at threads={threads}; "
                         f"2 frames ({dt1:.1f} s) at threads=1; " +
                         ("the reference package itself (baseline/_ref stereonorm 0.1.0: "
                          "estimate_normals_fixed + triangulate_grid + depth_laplacian "
                          "predicate) + scipy 8-connected labels" if kind == "reference" else
                          "oracle port of estimate_normals_fixed + triangulate_grid + ST labels")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Mpx/s", "n_gpus": world,
            "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
            "data": "synthetic: raycast street scene (SURVEY.md C3) + device N(0,0.2) noise",
            # the same config dict as the reference arm's line (same workload)
            "config": {"workload": WORKLOAD if args.pipeline == "full" else
                       "C3 2048x1024 street, fixed 9x9 pass",
                       "height": H, "width": W, "kernel": KSIZE},
            "config_detail": {"frames_per_gpu": B, "io": IO,
                              "parallelism": f"frame-batch dp{world}",
                              "l2": "inputs+outputs (15 GB/step) >> 126 MB L2, no flush needed"},
            "frames_per_sec_per_gpu": B / (ms_per_step / 1e3),
            "stages_ms_per_frame": {"fused_pass": fused_avg / B,
                                    "labels_incl_passable_bits": ccl_avg / B},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "fixed_square_kernel<4,float>",
                         "bytes_per_px": fused_bytes,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if pk.exists() else "fallback"},
            "e2e": e2e,
            "cpu_baseline": cpu,
            "configs": configs,
            "next_rows_us_per_frame": extras,
            "next_rows_roofline": extras_roof,
            "next_rows_cpu_us_per_frame": extras_cpu,
            # fused pass + (bits, tile, seam, resolve) per half batch: two
            # halves from 128 frames on (sn_ccl_labels_ws)
            "gpu_launches": args.steps * (1 + ((8 if B >= 128 else 4) if args.pipeline == "full" else 0)),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
