"""Per-source-line instructions executed + stall samples for one kernel of an ncu report."""
import collections, csv, io, subprocess, sys

rep, kf = sys.argv[1], sys.argv[2]
src = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kf}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
cur = None
agg = collections.defaultdict(lambda: [0, 0, ""])
for r in csv.reader(io.StringIO(out)):
    if len(r) == 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] in ("Line No", ""):
        continue
    try:
        k = (cur, int(r[0]))
        agg[k][0] += int(r[4])
        agg[k][1] += int(r[7]) if r[7] not in ("-", "") else 0
        agg[k][2] = r[1][:80]
    except ValueError:
        pass
tot_i = sum(v[1] for v in agg.values()) or 1
tot_s = sum(v[0] for v in agg.values()) or 1
print(f"total inst {tot_i}  samples {tot_s}")
for k in sorted(agg):
    v = agg[k]
    if (src is None or k[0] == src) and (v[1] > tot_i * 0.004 or v[0] > tot_s * 0.004):
        print(f"{k[0]}:{k[1]:4d} inst {100 * v[1] / tot_i:5.1f}%  samp {100 * v[0] / tot_s:5.1f}%  {v[2]}")
