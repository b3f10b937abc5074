"""Turn one GPU session's ncu outputs (gpurun_out/) into the committed summaries
under profiles/:

  profiles/launches_<tag>.csv       the launch list (gpu__time_duration.sum per launch)
  profiles/launches_<tag>.txt       per-kernel mean time and share of the step
  profiles/ncu_<name>_<tag>.txt     --set full summaries (tools/ncu_summary.py + hot lines)
  profiles/ncu_summary.json         per-launch DRAM traffic of the fused pass (bench.py's
                                    roofline.traffic) and per-frame CCL times

    python tools/make_profiles.py <tag> [frames_in_full_capture]
"""

import collections
import csv
import json
import shutil
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"


def launch_table(tag):
    src = OUT / f"launches_{tag}.csv"
    if not src.exists():
        return None
    shutil.copy(src, PROF / src.name)
    rows = list(csv.reader(open(src)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        unit = d.get("Metric Unit", "ns")
        v = v * {"ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
        agg.setdefault(d["Kernel Name"][:100], []).append(v)
    ours = {k: v for k, v in agg.items() if "sn::" in k}
    tot = sum(sum(v) for v in ours.values()) or 1.0
    lines = [f"launch list {src.name} (ncu --metrics gpu__time_duration.sum --clock-control none;"
             " cold-cache, serialised launches: compare SHARES, not absolute times)", ""]
    lines.append(f"{'launches':>8} {'mean us':>10} {'share':>7}  kernel")
    for k, v in sorted(ours.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"{len(v):8d} {sum(v) / len(v):10.1f} {100 * sum(v) / tot:6.1f}%  {k}")
    others = {k: v for k, v in agg.items() if "sn::" not in k}
    if others:
        lines += ["", "not ours (input synthesis outside the timed region):"]
        for k, v in others.items():
            lines.append(f"{len(v):8d} {sum(v) / len(v):10.1f}          {k}")
    (PROF / f"launches_{tag}.txt").write_text("\n".join(lines) + "\n")
    return {k: sum(v) / len(v) for k, v in ours.items()}


def raw_metrics(rep, kfilter):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv", "-k",
                          f"regex:{kfilter}"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for h, u, v in zip(hdr, units, r):
            d[h] = (v, u)
        res.append(d)
    return res


def num(d, key):
    v, u = d.get(key, ("nan", ""))
    v = float(v.replace(",", "")) if v not in ("", "n/a") else float("nan")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
             "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6,
             "ms": 1e-3, "s": 1.0}.get(u, 1.0)
    return v * scale


def full_summary(tag, name, kfilter, hot=None):
    rep = OUT / f"{name}_{tag}.ncu-rep"
    if not rep.exists():
        return None
    txt = subprocess.run([sys.executable, str(ROOT / "tools" / "ncu_summary.py"), str(rep),
                          kfilter] + ([hot, "25"] if hot else []), capture_output=True,
                         text=True).stdout
    (PROF / f"ncu_{name}_{tag}.txt").write_text(txt)
    return raw_metrics(rep, kfilter)


def main():
    tag = sys.argv[1]
    frames = int(sys.argv[2]) if len(sys.argv) > 2 else 256
    PROF.mkdir(exist_ok=True)
    launches = launch_table(tag)
    summ = {"tag": tag, "frames_per_launch_in_full_capture": frames}
    fused = full_summary(tag, "fused", "fixed_square", "fixed_square")
    if fused:
        d = fused[0]
        rd, wr = num(d, "dram__bytes_read.sum"), num(d, "dram__bytes_write.sum")
        t = num(d, "gpu__time_duration.sum")
        px = frames * 2048 * 1024
        summ["fused_pass"] = {
            "kernel": "fixed_square_kernel<4,float>",
            "dram_bytes_read": rd, "dram_bytes_write": wr,
            "dram_bytes_per_launch_at_c3": (rd + wr) * 256 / frames,
            "dram_bytes_per_px": (rd + wr) / px,
            "algorithmic_bytes_per_px": 28.0,
            "ncu_time_ms": t * 1e3,
            "dram_gbs_under_ncu": (rd + wr) / t / 1e9,
        }
    ccl = full_summary(tag, "ccl", "ccl_|passable_bits")
    if ccl:
        # from 128 frames on the labels run as two half batches (sn_ccl_labels_ws):
        # each predicate / labeller launch covers half the frames
        lf = frames // 2 if frames >= 128 else frames
        summ["ccl"] = {"frames_per_launch": lf}
        for d in ccl:
            name = d.get("Kernel Name", ("?", ""))[0][:60]
            summ["ccl"][name] = {"us_per_frame_under_ncu": num(d, "gpu__time_duration.sum") * 1e6 / lf,
                                 "dram_bytes_per_px": (num(d, "dram__bytes_read.sum") +
                                                       num(d, "dram__bytes_write.sum")) / (lf * 2048 * 1024)}
    if launches:
        summ["launch_list_mean_us"] = launches
    (PROF / "ncu_summary.json").write_text(json.dumps(summ, indent=1) + "\n")
    print(json.dumps(summ, indent=1))


if __name__ == "__main__":
    main()
