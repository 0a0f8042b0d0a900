"""Summarise an ncu report: key metrics + hottest SASS windows (needs -lineinfo build)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
W = int(sys.argv[2]) if len(sys.argv) > 2 else 64
kf = ["-k", f"regex:{sys.argv[3]}"] if len(sys.argv) > 3 else []
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"] + kf, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
d = dict(zip(rows[0], rows[2]))
keys = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__thread_inst_executed.sum"]
for k in keys:
    print(f"{k} = {d.get(k)}")
stalls = [k for k in d if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")]
for k in sorted(stalls, key=lambda k: -float(d[k] or 0))[:8]:
    print(f"{k.replace('smsp__average_warps_issue_stalled_', 'stall_')} = {d[k]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + kf, capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = next(k for k, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
data = [r for r in rows[hi + 1:] if r and r[0].startswith("0x")]
ia, ie, it = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"), hdr.index("Avg. Threads Executed")
tot = sum(int(r[ia] or 0) for r in data) or 1
totI = sum(int(r[ie] or 0) for r in data) or 1
win = {}
for k, r in enumerate(data):
    a = win.setdefault(k // W, [0, 0, k, 0.0])
    a[0] += int(r[ia] or 0)
    a[1] += int(r[ie] or 0)
    a[3] += int(r[ie] or 0) * float(r[it] or 0)
print(f"SASS lines {len(data)}; hottest {W}-instruction windows:")
for w, (s, i, k, th) in sorted(win.items(), key=lambda x: -x[1][0])[:10]:
    print(f"  @{k:6d} samples {100 * s / tot:5.1f}%  inst {100 * i / totI:5.1f}%  threads {th / max(i, 1):4.1f}  {data[k][1][:48]}")
