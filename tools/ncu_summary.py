"""Summarise an ncu report: per-kernel time, DRAM bytes, throughput, stalls, hot lines."""
import csv, io, subprocess, sys

def raw(rep, kfilter=None):
    args = ["ncu", "-i", rep, "--page", "raw", "--csv"]
    if kfilter: args += ["-k", f"regex:{kfilter}"]
    out = subprocess.run(args, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'launch__registers_per_thread',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 'launch__occupancy_limit_shared_mem',
        'launch__occupancy_limit_registers', 'lts__t_bytes.sum']

def hot_lines(rep, kfilter, n=20):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kfilter}",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    cur = None; agg = []
    for r in csv.reader(io.StringIO(out)):
        if len(r) == 2 and r[0] == 'File Path': cur = r[1].split('/')[-1]; continue
        if len(r) < 8 or r[0] in ('Line No', ''): continue
        try: agg.append((int(r[4]), int(r[7]) if r[7] not in ('-', '') else 0, cur, r[0], r[1][:90]))
        except ValueError: pass
    tot = sum(a[0] for a in agg) or 1
    for a in sorted(agg, reverse=True)[:n]:
        print(f"   {a[0]:6d} {100*a[0]/tot:5.1f}% inst={a[1]:10d} {a[2]}:{a[3]} {a[4]}")

if __name__ == "__main__":
    rep = sys.argv[1]; kf = sys.argv[2] if len(sys.argv) > 2 else None
    hdr, units, rows = raw(rep, kf)
    for r in rows:
        print("===", r[hdr.index('Kernel Name')][:90])
        for w in WANT:
            if w in hdr: print(f"   {w} = {r[hdr.index(w)]} {units[hdr.index(w)]}")
        st = sorted(((float(r[i].replace(',', '')), hdr[i]) for i in range(len(hdr))
                     if hdr[i].startswith('smsp__pcsamp_warps_issue_stalled') and not hdr[i].endswith('not_issued')
                     and r[i] not in ('', 'n/a')), reverse=True)[:8]
        print("   stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_','')}={v:.0f}" for v, k in st))
    if len(sys.argv) > 3:
        hot_lines(rep, sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 20)
