"""Runs tools/alu_peak (issue-rate microbenchmarks) on the B200 and writes the
measured ALU / fp64 roofline denominators to profiles/alu_peak_r02.json.

  python tools/alu_peak.py [--ncu]        # on the GPU box (gpurun)

Timing: the binary's CUDA-event best-of-N per kernel, with nvidia-smi SM
clocks sampled during the run.  Instruction counts: one ncu pass
(`smsp__inst_executed.sum` and the per-pipe counters) over the same binary, so
the issue rates are SASS warp instructions per second, per SM per clock.
"""
import csv
import io
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tools", "alu_peak")
SRC = os.path.join(ROOT, "tools", "alu_peak.cu")
OUT = os.path.join(ROOT, "profiles", "r02", "alu_peak.json")
METRICS = ["smsp__inst_executed.sum", "smsp__thread_inst_executed.sum", "sm__inst_executed_pipe_alu.sum",
           "sm__inst_executed_pipe_fma.sum", "sm__inst_executed_pipe_fp64.sum", "gpu__time_duration.sum"]
NAMES = {"k_iadd": "iadd", "k_mix": "mix", "k_imax64": "imax64", "k_dcell": "dcell", "k_dadd": "dadd"}


def build():
    if not os.path.exists(BIN) or os.path.getmtime(BIN) < os.path.getmtime(SRC):
        subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-O3", "-std=c++17", "-gencode",
                               "arch=compute_100a,code=sm_100a", "-lineinfo", SRC, "-o", BIN])


def clocks_during(cmd):
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm", "--format=csv,noheader,nounits",
                            "-lms", "50", "-i", "0"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    time.sleep(0.3)
    out = subprocess.check_output(cmd, text=True)
    smi.terminate()
    s, _ = smi.communicate(timeout=10)
    sm = []
    mx = 0.0
    for line in s.strip().splitlines():
        try:
            a, b = [float(x) for x in line.split(",")]
        except ValueError:
            continue
        sm.append(a)
        mx = max(mx, b)
    loaded = [x for x in sm if x > 0.5 * mx] or sm
    return out, (statistics.median(loaded) if loaded else None), mx


def ncu_counts():
    out = subprocess.run(["ncu", "--metrics", ",".join(METRICS), "--clock-control", "none", "--csv",
                          BIN, "1"], capture_output=True, text=True)
    with open(os.path.join(ROOT, "gpurun_out", "alu_peak_ncu.csv"), "w") as f:
        f.write(out.stdout + "\n" + out.stderr)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    h0 = next(k for k, r in enumerate(rows) if "Metric Name" in r)
    hdr, rows = rows[h0], rows[h0:]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    res = {}
    for r in rows[1:]:
        if len(r) != len(hdr):
            continue
        k = NAMES.get(r[ki].split("(")[0].strip())
        if not k:
            continue
        v = float(r[vi].replace(",", ""))
        res.setdefault(k, {})[r[mi]] = v   # last launch wins (identical launches)
    return res


def main():
    build()
    out, sm_mhz, sm_max = clocks_during([BIN, "30"])
    js = json.loads(out)
    res = {"what": "issue-rate microbenchmarks (tools/alu_peak.cu): NCH=8 independent chains per thread, "
                   "grid 148x8 blocks x 256 threads, best-of-30 CUDA-event time per kernel",
           "sm_mhz_median_under_load": sm_mhz, "sm_max_mhz": sm_max, "sms": js["sms"], "kernels": {}}
    counts = ncu_counts() if "--ncu" in sys.argv else {}
    clk = (sm_mhz or sm_max) * 1e6
    for k, v in js["kernels"].items():
        e = dict(v)
        c = counts.get(k)
        if c:
            inst = c["smsp__inst_executed.sum"]
            s = v["ms"] * 1e-3
            e["warp_inst"] = inst
            e["warp_inst_per_s"] = inst / s
            e["warp_inst_per_sm_clk"] = inst / s / js["sms"] / clk
            e["thread_inst_per_s"] = c["smsp__thread_inst_executed.sum"] / s
            e["pipe_alu_frac"] = c["sm__inst_executed_pipe_alu.sum"] / inst
            e["pipe_fma_frac"] = c["sm__inst_executed_pipe_fma.sum"] / inst
            e["pipe_fp64_frac"] = c["sm__inst_executed_pipe_fp64.sum"] / inst
            e["sass_inst_per_unit"] = c["smsp__thread_inst_executed.sum"] / (v["units_per_s"] * s)
        res["kernels"][k] = e
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    with open(OUT, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
