"""Summarise gpurun_out/ ncu outputs into profiles/ (launch list shares, DRAM traffic,
issue / warp utilisation of the dominant kernel).  Usage: summarize_profiles.py <round tag>"""
import csv
import io
import json
import os
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
go = os.path.join(root, "gpurun_out")
prof = os.path.join(root, "profiles")

rows = [r for r in csv.reader(open(os.path.join(go, "launches.csv"))) if len(r) > 10]
hdr, data = rows[0], rows[1:]
ik, im, iv, iid = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
launch = {}
for r in data:
    launch.setdefault(int(r[iid]), {"kernel": r[ik].split("(")[0].replace("void ", "")})[r[im]] = float(r[iv].replace(",", ""))
ids = sorted(launch)
# prof_sweep runs 2 sweeps: take the second (warm) one = second half of the launches
half = ids[len(ids) // 2:]
tot_ns = sum(launch[i]["gpu__time_duration.sum"] for i in half)
dram = sum(launch[i].get("dram__bytes_read.sum", 0) + launch[i].get("dram__bytes_write.sum", 0) for i in half)
winst = sum(launch[i].get("smsp__inst_executed.sum", 0) for i in half)
tinst = sum(launch[i].get("smsp__thread_inst_executed.sum", 0) for i in half)
kern = []
for i in half:
    L = launch[i]
    kern.append({"kernel": L["kernel"], "us": round(L["gpu__time_duration.sum"] / 1e3, 1),
                 "share_of_serialised_sum": round(L["gpu__time_duration.sum"] / tot_ns, 3),
                 "dram_MB": round((L.get("dram__bytes_read.sum", 0) + L.get("dram__bytes_write.sum", 0)) / 1e6, 2),
                 "warp_inst_M": round(L.get("smsp__inst_executed.sum", 0) / 1e6, 1),
                 "issue_active_pct": L.get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                 "warps_active_pct": L.get("sm__warps_active.avg.pct_of_peak_sustained_active")})


def raw(rep, regex):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", f"regex:{regex}"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(out)))
    res = []
    for r in rr[2:]:
        d = dict(zip(rr[0], r))
        res.append(d)
    return res


full = {}
keys = ["gpu__time_duration.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "dram__bytes_write.sum.per_second"]
for rep, rx in (("prof_pipe4.ncu-rep", "k_pipe"), ("prof_phases.ncu-rep", "k_")):
    p = os.path.join(go, rep)
    if os.path.exists(p):
        for d in raw(p, rx):
            name = d.get("Kernel Name", "?").split("(")[0].replace("void ", "")
            full[name] = {k: d.get(k) for k in keys}
            st = sorted([k for k in d if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")],
                        key=lambda k: -float(d[k] or 0))[:5]
            full[name]["top_stalls_per_issue"] = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): d[k] for k in st}
summary = {"round": tag, "workload": "config 2 full sweep (873192 candidates) -> top-16, one hsim_topk call",
           "how": "ncu --metrics ... --clock-control none (cold, serialised: shares, not absolutes); second of two sweeps",
           "serialised_sum_us": round(tot_ns / 1e3, 1), "sweep_dram_bytes": int(dram),
           "sweep_warp_inst": int(winst), "sweep_thread_inst": int(tinst), "kernels": kern, "full_captures": full}
os.makedirs(prof, exist_ok=True)
json.dump(summary, open(os.path.join(prof, f"ncu_summary_{tag}.json"), "w"), indent=1)
json.dump({"sweep_dram_bytes": int(dram) or None, "sweep_warp_inst": int(winst), "sweep_thread_inst": int(tinst) or None,
           "config": 2, "round": tag}, open(os.path.join(prof, "ncu_summary.json"), "w"), indent=1)
subprocess.run(["cp", os.path.join(go, "launches.csv"), os.path.join(prof, f"launches_{tag}.csv")])
for k in kern:
    print(k)
print("sweep dram bytes", dram)
for n, f in full.items():
    print(n, {k.split("__")[-1][:40]: v for k, v in f.items() if k != "top_stalls_per_issue"}, f["top_stalls_per_issue"])
