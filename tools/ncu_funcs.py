"""Attribute ncu SASS samples/instructions to call targets (noinline functions) of a kernel."""
import csv
import io
import re
import subprocess
import sys

rep, so, kern = sys.argv[1], sys.argv[2], sys.argv[3]
sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
blk = sass[sass.index("Function : " + kern):]
nxt = blk.find("Function : ", 20)
blk = blk if nxt < 0 else blk[:nxt]
targets = sorted({int(t, 16) for t in re.findall(r"CALL\.REL\.NOINC (0x[0-9a-f]+)", blk)})
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr, data = rows[1], rows[2:]
ia, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
cols = [c for c in ("stall_no_inst", "stall_wait", "stall_short_sb", "stall_long_sb", "stall_branch_resolving", "stall_selected") if c in hdr]
ic = [hdr.index(c) for c in cols]
base = int(data[0][0], 16)
agg = {}
for r in data:
    off = int(r[0], 16) - base
    f = max([t for t in targets if t <= off], default=0)
    a = agg.setdefault(f, [0, 0, off] + [0] * len(ic))
    a[0] += int(r[ia] or 0)
    a[1] += int(r[ie] or 0)
    for q, j in enumerate(ic):
        a[3 + q] += int(r[j] or 0)
tot = sum(a[0] for a in agg.values()) or 1
totI = sum(a[1] for a in agg.values()) or 1
print("stall columns:", cols)
for f, a in sorted(agg.items(), key=lambda x: -x[1][0]):
    s, i = a[0], a[1]
    st = " ".join(f"{100 * v / tot:5.1f}" for v in a[3:])
    print(f"fn@0x{f:06x}  samples {100 * s / tot:5.1f}%  inst {100 * i / totI:5.1f}%  | {st}")
