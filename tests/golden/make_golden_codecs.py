"""Golden decoder vectors from the REFERENCE readers (formats.py:55-162).

Run in the build container (reads /root/reference):

    python tests/golden/make_golden_codecs.py

Writes ``codec_cases.npz``:
  * pfm_<name>:  file bytes + the reference's read_pfm / read_pfm_normals
                 values and mask (little/big endian, 1/3 channels, odd widths,
                 NaN/inf samples, extra header whitespace);
  * pfmerr_<i>:  malformed files + the reference's FormatError message;
  * png_<name>:  16-bit PNG bytes, (scale, invalid) + read_disparity_png16's
                 values and mask;
  * fused_<name>: a quantised street crop as PNG16 + estimate_normals_fixed
                 and triangulate_grid on the reference's decoded field.
"""

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(Path(__file__).resolve().parent))
import stereonorm as sn  # noqa: E402
from stereonorm import formats  # noqa: E402

from make_golden import street_scene  # noqa: E402

OUT = Path(__file__).resolve().parent
rng = np.random.default_rng(77)
store = {}


def u8(b):
    return np.frombuffer(bytes(b), dtype=np.uint8)


def pfm_bytes(grid, big_endian, channels, header=None):
    h, w = grid.shape[:2]
    magic = "PF" if channels == 3 else "Pf"
    hdr = header or f"{magic}\n{w} {h}\n{'1.0' if big_endian else '-1.0'}\n"
    return hdr.encode("ascii") + grid[::-1].astype(">f4" if big_endian else "<f4").tobytes()


# ---- PFM
pfm_names = []
for name, h, w, ch, be, hdr in [("le_16x12", 12, 16, 1, False, None),
                                ("be_16x12", 12, 16, 1, True, None),
                                ("le_odd", 7, 13, 1, False, None),
                                ("be_odd", 9, 5, 1, True, None),
                                ("rgb_le", 6, 8, 3, False, None),
                                ("rgb_be", 5, 7, 3, True, None),
                                ("ws_hdr", 3, 5, 1, False, "Pf \n 5   3\n-2.5\n"),
                                ("be_scale", 4, 4, 1, True, "Pf\n4 4\n3.0\n")]:
    shape = (h, w, 3) if ch == 3 else (h, w)
    g = rng.normal(10, 5, shape).astype(np.float32)
    flat = g.reshape(-1)
    flat[rng.random(flat.size) < 0.1] = np.nan
    flat[3] = np.inf
    flat[5] = -np.inf
    flat[7] = -0.0
    flat[8] = 1e-40  # subnormal survives the byte path
    data = pfm_bytes(g, be, ch, hdr)
    f = formats.read_pfm_normals(data) if ch == 3 else formats.read_pfm(data)
    p = f"pfm_{name}__"
    store[p + "bytes"] = u8(data)
    store[p + "values"] = f.vectors if ch == 3 else f.values
    store[p + "mask"] = f.mask
    store[p + "channels"] = np.array(ch)
    pfm_names.append(name)

bad = [b"", b"Pf\n4 4", b"PX\n4 4\n-1.0\n" + b"\0" * 64, b"Pf\n4 x\n-1.0\n",
       b"Pf\n0 4\n-1.0\n", b"Pf\n4 4\n0.0\n", b"Pf\n4 4\n-1.0\n" + b"\0" * 60,
       b"Pf\n4 4\n-1.0", b"PF\n2 2\n-1.0\n" + b"\0" * 48]
msgs = []
for i, b in enumerate(bad):
    try:
        formats.read_pfm(b)
        raise SystemExit(f"malformed case {i} was accepted")
    except formats.FormatError as exc:
        msgs.append(str(exc))
    store[f"pfmerr_{i}__bytes"] = u8(b)
store["pfmerr_msgs"] = np.array(msgs)

# ---- PNG16
png_names = []
raw_cases = []
r = rng.integers(0, 65536, (23, 29)).astype(np.uint16)
r[0, :5] = [0, 1, 2, 65535, 65534]
raw_cases += [("raw_s256_i0", r, 256.0, 0), ("raw_s100_i0", r, 100.0, 0),
              ("raw_s256_i65535", r, 256.0, 65535), ("raw_s3_i1", r, 3.0, 1),
              ("raw_neg", r, -64.0, 0), ("raw_noinv", r, 256.0, 70000)]
for name, raw, scale, inv in raw_cases:
    from PIL import Image
    import io
    buf = io.BytesIO()
    Image.fromarray(raw).save(buf, format="PNG")
    data = buf.getvalue()
    f = formats.read_disparity_png16(data, scale, inv)
    p = f"png_{name}__"
    store[p + "bytes"] = u8(data)
    store[p + "scale"] = np.array(scale)
    store[p + "invalid"] = np.array(inv)
    store[p + "raw"] = raw
    store[p + "values"] = f.values
    store[p + "mask"] = f.mask
    png_names.append(name)

# ---- fused PNG16 -> oriented points
fused_names = []
rig_s, gts = street_scene(256, 128, fx=256.0)
noisy = sn.add_gaussian_noise(gts.disparity, 0.3, seed=11)
for name, scale, k in [("street_s256_k9", 256.0, 9), ("street_s100_k5", 100.0, 5),
                       ("street_s256_k15", 256.0, 15)]:
    data = formats.write_disparity_png16(noisy, scale, 0)
    field = formats.read_disparity_png16(data, scale, 0)
    nf = sn.estimate_normals_fixed(field, rig_s, sn.build_kernels(sn.KernelSpec.square(k)))
    pts = sn.triangulate_grid(field, rig_s)
    p = f"fused_{name}__"
    store[p + "bytes"] = u8(data)
    store[p + "scale"] = np.array(scale)
    store[p + "k"] = np.array(k)
    store[p + "rig"] = np.array([rig_s.fx, rig_s.fy, rig_s.u0, rig_s.v0, rig_s.baseline])
    store[p + "normals"] = nf.vectors
    store[p + "nmask"] = nf.mask
    store[p + "points"] = pts
    fused_names.append(name)

store["pfm_names"] = np.array(pfm_names)
store["png_names"] = np.array(png_names)
store["fused_names"] = np.array(fused_names)
np.savez_compressed(OUT / "codec_cases.npz", **store)
print("wrote", OUT / "codec_cases.npz", len(pfm_names), len(bad), len(png_names),
      len(fused_names))
