"""Per-kernel table of an ncu launch list (the second of the profiled sweeps)."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv")) if len(r) > 10]
hdr, data = rows[0], rows[1:]
ik, im, iv, iid = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
L = {}
for r in data:
    L.setdefault(int(r[iid]), {"k": r[ik].split("(")[0].replace("void ", "")})[r[im]] = float(r[iv].replace(",", ""))
ids = sorted(L)
half = ids[len(ids) // 2:]
tot = sum(L[i]["gpu__time_duration.sum"] for i in half)
print(f"{len(half)} launches, serialised sum {tot / 1e3:.1f} us")
for i in half:
    d = L[i]
    print(f"{d['k'][:40]:40s} {d['gpu__time_duration.sum'] / 1e3:8.1f} us  {d.get('smsp__inst_executed.sum', 0) / 1e6:7.1f} Minst  "
          f"issue {d.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):5.1f}%  warps {d.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):5.1f}%")
