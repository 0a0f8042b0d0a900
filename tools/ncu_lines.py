"""Per-CUDA-source-line stall samples / instructions of one kernel in an ncu report
(`--print-source cuda,sass`).  Usage: ncu_lines.py <rep> <kernel regex> [top]"""
import csv
import io
import subprocess
import os
import sys

rep, rx = sys.argv[1], sys.argv[2]
SORTI = int(os.environ.get("SORTI", "0"))
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{rx}"],
                     capture_output=True, text=True).stdout
fname, line, src = "?", "?", ""
agg = {}
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0] not in ("", "-"):
        line, src = r[0], r[1]
        continue
    if not r[2].startswith("0x"):
        continue
    a = agg.setdefault((fname, line), [0, 0, src])
    a[0] += int(r[4] or 0)
    a[1] += int(r[7] or 0)
ts = sum(v[0] for v in agg.values()) or 1
ti = sum(v[1] for v in agg.values()) or 1
print(f"total samples {ts}, warp instructions {ti}")
for (f, l), (s, i, src) in sorted(agg.items(), key=lambda x: -x[1][SORTI])[:top]:
    print(f"{f}:{l:>5} stall {100 * s / ts:5.1f}%  inst {100 * i / ti:5.1f}%  {src.strip()[:90]}")
