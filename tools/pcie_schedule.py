"""PCIe schedule probe for the host pipeline's copies (no compute): a 64-frame C3
step moves 8.4 MB/frame host->device and 58.7 MB/frame device->host, in the
pipeline's chunks (1, 2, 4, then 8 frames).  Times, with pinned buffers:
  d2h only     the D2H chunks back to back
  h2d only     the H2D chunks back to back
  pipeline     H2D of chunk c queued when the D2H of chunk c-3 is done (about
               what sn_pipeline_host's slot events allow), D2H on its own stream
  fine         each chunk's H2D split into 8 pieces, piece j queued after the
               j-th eighth of an earlier chunk's D2H (the H2D spread thin)
  serial       all H2D, then all D2H
"""
import sys
import time

import torch

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
PX = 1024 * 2048
IN_F, OUT_F = PX * 4, PX * 28
sizes = []
f = 0
while f < B:
    n = min(B - f, 8 if len(sizes) >= 3 else 1 << len(sizes))
    sizes.append(n)
    f += n
h_in = torch.empty(B * IN_F, dtype=torch.uint8).pin_memory()
h_out = torch.empty(B * OUT_F, dtype=torch.uint8).pin_memory()
d_in = torch.empty(B * IN_F, dtype=torch.uint8, device="cuda")
d_out = torch.empty(B * OUT_F, dtype=torch.uint8, device="cuda")
s_h = torch.cuda.Stream()
s_d = torch.cuda.Stream()


def chunks(per):
    o = 0
    for n in sizes:
        yield o * per, n * per
        o += n


def d2h_only():
    with torch.cuda.stream(s_d):
        for o, n in chunks(OUT_F):
            h_out[o:o + n].copy_(d_out[o:o + n], non_blocking=True)


def h2d_only():
    with torch.cuda.stream(s_h):
        for o, n in chunks(IN_F):
            d_in[o:o + n].copy_(h_in[o:o + n], non_blocking=True)


def pipeline(pieces=1, lag=3):
    ins = list(chunks(IN_F))
    outs = list(chunks(OUT_F))
    marks = []  # events after each D2H piece
    for c in range(len(sizes)):
        # H2D of chunk c, gated on the D2H of chunk c - lag
        o, n = ins[c]
        step = (n + pieces - 1) // pieces
        for j in range(pieces):
            k = (c - lag) * pieces + j
            if k >= 0 and k < len(marks):
                s_h.wait_event(marks[k])
            with torch.cuda.stream(s_h):
                a = o + j * step
                b = min(o + n, a + step)
                if a < b:
                    d_in[a:b].copy_(h_in[a:b], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(s_h)
        s_d.wait_event(ev)
        o, n = outs[c]
        step = (n + pieces - 1) // pieces
        for j in range(pieces):
            with torch.cuda.stream(s_d):
                a = o + j * step
                b = min(o + n, a + step)
                if a < b:
                    h_out[a:b].copy_(d_out[a:b], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s_d)
                marks.append(e)


def serial():
    h2d_only()
    s_d.wait_stream(s_h)
    d2h_only()


def timeit(fn, n=3):
    best = 1e9
    for _ in range(n + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best * 1e3


print("chunks (frames):", sizes)
for name, fn in [("d2h only", d2h_only), ("h2d only", h2d_only), ("pipeline", pipeline),
                 ("fine x8", lambda: pipeline(8)), ("fine x8 lag 1", lambda: pipeline(8, 1)),
                 ("serial", serial), ("d2h only", d2h_only), ("pipeline", pipeline)]:
    print(f"{name:14s} {timeit(fn):8.2f} ms")
