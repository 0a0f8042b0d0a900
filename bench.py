"""Benchmark: simulated candidate configurations per second (BASELINE.json metric)
on the hetero Llama-2-7B sweep (BASELINE config 2: 16xA100 + 16xH100,
873,192 candidates), 1..N B200s, plus the ALU-issue roofline fraction.

One step = one full sweep of the config-2 space -> global top-k (hsim_topk on
each rank's block-cyclic shard; for N > 1 one NCCL all_gather of the k-entry
lists and the hsim_merge_topk kernel).  Total work is fixed as N grows
("scaling": "strong").  L2 is flushed (a 512 MiB write) between timed steps,
outside the CUDA-event intervals.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

--impl reference times the CPU oracle (the paper-derived reference of this
tier) on the host cores, on a bounded sample of the same
workload per step; rank 0 only.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import hsim_inputs as H  # noqa: E402

METRIC = "simulated configs/sec, 1/2/4/8 B200, hetero Llama-7B sweep; % ALU-issue peak"
CONFIG = 2
TOPK = 16
# ALU-issue roofline: 148 SMs x 4 SMSPs x 32 lanes x SM clock
SMS, LANES_PER_SM = 148, 128
OPS_PER_CELL = 8  # int32-equivalent ops per 1F1B max-plus cell


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=CONFIG)
    ap.add_argument("--k", type=int, default=TOPK)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--mem-check", action="store_true",
                    help="SURVEY 8(f) f2 row: prune candidates over device memory (status -3, DESIGN M.1)")
    ap.add_argument("--sync-overlap", action="store_true",
                    help="SURVEY 8(f) f1 row: gradient sync overlapped with the backward (DESIGN S.1)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                       "-lms", "100", "-i", str(self.gpu)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def overhead_ops(sim, first, n, blk, stride, world, sync_units=-1):
    """SURVEY §8(d) per-candidate non-cell work: 50 ops per stage (partition +
    stage sums), 26 per gradient-sync segment (J = sum P_c - C + 1, the most the
    common refinement can have), 100 for the decode -- summed over this rank's
    candidates template by template (host decode of each template's first
    candidate; outside the timed region).  sync_units >= 0: the sweep pruned the
    sync (hsim_last_sync_units: sum of J over the candidates whose sync ran),
    so only those segments are counted."""
    tot = 0
    nt = sim.n_templates()
    bounds = [sim.template_first(k) for k in range(nt + 1)]
    ranges = [(first, first + n)] if world == 1 else \
        [(b0, min(b0 + blk, sim.space_size())) for b0 in range(first, sim.space_size(), stride)]
    import bisect
    for lo, hi in ranges:
        k = bisect.bisect_right(bounds, lo) - 1
        while k < nt and bounds[k] < hi:
            cnt = min(hi, bounds[k + 1]) - max(lo, bounds[k])
            d = sim.decode(bounds[k])
            sp = sum(len(c["stages"]) for c in d["classes"])
            J = sp - len(d["classes"]) + 1
            tot += cnt * (50 * sp + (26 * J if sync_units < 0 else 0) + 100)
            k += 1
    return tot + (26 * sync_units if sync_units >= 0 else 0)


def cpu_baseline(cfg, seconds=15.0):
    """The oracle as it stands, on all host cores, on a seeded sample of the
    workload sized to ~`seconds` of wall time (rank 0, N=1 only)."""
    import oracle
    o = oracle.Oracle(cfg, compact=True)
    cores = os.cpu_count() or 1
    N = o.space_size()
    cal = H.sample_indices(N, 4 * cores, seed=1)
    t = time.perf_counter()
    o.eval_many(cal, threads=cores)
    rate = len(cal) / max(time.perf_counter() - t, 1e-6)
    n = int(min(max(rate * seconds, 64), N))
    idx = H.sample_indices(N, n, seed=H.PARITY_SEED)
    t = time.perf_counter()
    o.eval_many(idx, threads=cores)
    dt = time.perf_counter() - t
    return {"value": round(len(idx) / dt, 3), "unit": "configs/s", "cores": cores, "kind": "oracle",
            "sample": f"{len(idx)} seeded (splitmix64 0x5EED2508) uniform candidates of the {N}-candidate "
                      f"{cfg['name']} space, oracle/oracle.cpp in its compact mode (event-driven 1F1B, one pipeline "
                      f"per sub-class, closed-form ring steps; equal to the literal mode by tests), {dt:.1f} s wall"}


def workload(a):
    cfg = H.get(a.config)
    if a.mem_check:
        cfg = H.with_mem_check(cfg)
    if a.sync_overlap:
        cfg = H.with_sync_overlap(cfg)
    return cfg


def run_reference(a):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle
    cfg = workload(a)
    o = oracle.Oracle(cfg, compact=True)
    cores = os.cpu_count() or 1
    N = o.space_size()
    per_step = max(4096, 2048 * cores)  # bounded sample per step (~0.05-0.2 s of host work)
    times = []
    for s in range(a.warmup + a.steps):
        idx = H.sample_indices(N, per_step, seed=H.PARITY_SEED + s)
        t = time.perf_counter()
        o.eval_many(idx, threads=cores)
        dt = time.perf_counter() - t
        if s >= a.warmup:
            times.append((len(idx), dt))
    cands = sum(c for c, _ in times)
    tot = sum(d for _, d in times)
    v = cands / tot
    line = {"metric": METRIC, "value": round(v, 3), "unit": "configs/s", "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": round(1e3 * tot / a.steps, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic", "impl": "reference",
            "config": {"workload": cfg["name"], "n_candidates": N,
                       "sample_per_step": per_step, "what": "CPU oracle (oracle/oracle.cpp, compact mode) on host cores"},
            "cpu_baseline": {"value": round(v, 3), "unit": "configs/s", "cores": cores, "kind": "oracle",
                             "sample": f"{per_step} seeded candidates per step x {a.steps} steps"},
            "e2e": {"value": round(v, 3), "unit": "configs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(a):
    import torch
    import torch.distributed as dist
    from paper_2508_05370_b200 import Sim, build as pbuild
    from paper_2508_05370_b200.sweep import shard, sweep

    rank, world, local = dist_env()
    assert world == a.gpus or world == 1, "launch with torchrun --nproc-per-node N for --gpus N > 1"
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if rank == 0:
        pbuild.build()
    if world > 1:
        dist.barrier()
    cfg = workload(a)
    sim = Sim(cfg)
    N = sim.space_size()
    first, n, blk, stride = shard(N, rank, world)
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    out = (torch.empty(a.k, dtype=torch.int64, device=dev), torch.empty(a.k, dtype=torch.int64, device=dev))

    def step():
        return sweep(sim, a.k, out=out)

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    # algorithmic work of this rank's shard: exact 1F1B cell count
    if world == 1:
        cells = sim.count_cells(0, N)
    else:
        cells = 0
        for b0 in range(first, N, stride):
            cells += sim.count_cells(b0, min(blk, N - b0))
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    clocks = Clocks(local if world > 1 else int(os.environ.get("CUDA_VISIBLE_DEVICES", "0").split(",")[0] or 0))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    for s in range(a.steps):
        flush.fill_(s & 0xFF)          # L2 flush between timed steps (not inside the events)
        if world > 1:                  # every rank starts the step together: barrier -> merged top-k
            dist.barrier()
            torch.cuda.synchronize()
        evs[s][0].record(stream)
        step()
        evs[s][1].record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    tot_ms = sum(ms)
    t_max = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    tot_ms = float(t_max.item())
    launches_per_step = sim.last_launch_count() + (1 if world > 1 else 0)
    value = N * a.steps / (tot_ms / 1e3)

    # roofline of the sweep: SURVEY §8(d)'s per-unit figures --
    # 8 int32-equivalent ops per EXECUTED 1F1B cell (the steady-regime jumps
    # skip cells; skipped cells are not counted) + per candidate ~50 ops per
    # stage (partition + stage sums), ~26 per sync segment (J <= sum P - C + 1),
    # ~100 for the decode -- over the ALU issue peak
    pk = peaks()
    sm_max = float(pk.get("sm_max_mhz", 1965.0))
    peak_gops = SMS * LANES_PER_SM * sm_max * 1e6 / 1e9
    my_ms = sum(ms) / a.steps
    sweep(sim, a.k, out=out)  # (untimed) the sync work the pruned sweep executes
    over = overhead_ops(sim, first, n, blk, stride, world, sim.last_sync_units())
    ops = OPS_PER_CELL * cells + over
    achieved = ops / (my_ms / 1e3) / 1e9
    traffic, issue = None, None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                js = json.load(f)
            if js.get("config") == a.config and world == 1 and not (a.mem_check or a.sync_overlap):
                traffic = js.get("sweep_dram_bytes")
                wi = js.get("sweep_warp_inst")
                if wi:  # ncu warp instructions of one sweep / (live sweep time x issue slots)
                    rate = wi / (my_ms / 1e3) / 1e9
                    issue = {"achieved": round(rate, 1), "peak": round(SMS * 4 * sm_max * 1e6 / 1e9, 1),
                             "unit": "Gwarp-inst/s", "frac": round(rate / (SMS * 4 * sm_max * 1e-3), 4),
                             "from": "profiles/ncu_summary.json sweep_warp_inst (ncu launch list of one sweep) / "
                                     "this run's mean sweep time; peak = 148 SMs x 4 schedulers x clock"}
        except (OSError, ValueError):
            traffic = None

    # e2e: explicit candidate list from pinned host memory -> eval -> results back to pinned host
    e2e = None
    if not a.no_e2e:
        idx_host = torch.arange(first, first + n, dtype=torch.int64) if world == 1 else \
            torch.tensor([first + (t // blk) * stride + t % blk for t in range(n)], dtype=torch.int64)
        idx_host = idx_host.pin_memory()
        res_host = torch.empty(n, dtype=torch.int64).pin_memory()
        e_steps = max(3, min(a.steps, 50))
        for s in range(3):
            sim.eval_host(idx_host, res_host)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if world > 1:
            dist.barrier()
        e0.record(stream)
        for s in range(e_steps):
            sim.eval_host(idx_host, res_host)   # chunked: H2D / eval / D2H overlapped
        e1.record(stream)
        torch.cuda.synchronize()
        et = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": round(N * e_steps / (float(et.item()) / 1e3), 1), "unit": "configs/s",
               "h2d_bytes_per_step": 8 * N, "d2h_bytes_per_step": 8 * N,
               "what": "Sim.eval_host: explicit index list in pinned host memory -> hsim_eval_batch in 2 chunks "
                       "-> int64 results in pinned host memory, H2D / compute / D2H overlapped on streams, every step"}

    # e2e of the sweep call itself: hsim_topk over the range (its inputs are the
    # descriptors, resident since create, and the range bounds) + the top-k read
    # back to pinned host memory every step
    e2e_sweep = None
    if not a.no_e2e:
        th = torch.empty(2 * a.k, dtype=torch.int64).pin_memory()
        for _ in range(3):
            t_, i_ = sweep(sim, a.k, out=out)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_steps = max(3, min(a.steps, 50))
        e0.record(stream)
        for _ in range(e_steps):
            t_, i_ = sweep(sim, a.k, out=out)
            th[:a.k].copy_(t_, non_blocking=True)
            th[a.k:].copy_(i_, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize()
        et = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e_sweep = {"value": round(N * e_steps / (float(et.item()) / 1e3), 1), "unit": "configs/s",
                     "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 16 * a.k,
                     "what": "Sim.topk over the whole range (the call `value` times) with the global top-k copied to "
                             "pinned host memory every step, back to back, no L2 flush"}

    # the same sweep without the pruned sync (every candidate's sync computed):
    # the comparison the pruning is judged against
    unpruned = None
    if world == 1:
        sim.set_prune(False)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        ums = []
        for s in range(min(a.steps, 50)):
            flush.fill_(s & 0xFF)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            torch.cuda.synchronize()
            ums.append(e0.elapsed_time(e1))
        sim.set_prune(True)
        um = sum(ums) / len(ums)
        unpruned = {"value": round(N / (um / 1e3), 1), "ms_per_step": round(um, 4), "steps": len(ums),
                    "what": "hsim_set_prune(0): the same full sweep -> top-k with every candidate's gradient sync "
                            "computed (K_sync); `value` computes it only where T0 can still enter the top-k"}

    # the same sweep with one 1F1B run per (candidate, class) instead of per
    # distinct class pipeline: the comparison the dedupe is judged against
    no_dedup = None
    if world == 1 and sim.dedup_active():
        sim.set_dedup(False)
        cells_off = sim.count_cells(0, N)
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        dms = []
        for s in range(min(a.steps, 50)):
            flush.fill_(s & 0xFF)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            torch.cuda.synchronize()
            dms.append(e0.elapsed_time(e1))
        sim.set_dedup(True)
        dm = sum(dms) / len(dms)
        no_dedup = {"value": round(N / (dm / 1e3), 1), "ms_per_step": round(dm, 4), "steps": len(dms),
                    "cells_per_launch": cells_off,
                    "what": "hsim_set_dedup(0): the same full sweep -> top-k with the 1F1B recurrence run once per "
                            "(candidate, class) instead of once per distinct class pipeline (DESIGN.md §5); exact "
                            "either way, `cells_per_launch` counts what executes"}

    # measured issue peaks (tools/alu_peak.cu microbenchmarks, profiles/r02/alu_peak.json)
    measured = None
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "alu_peak.json")) as f:
            ap = json.load(f)["kernels"]
        measured = {"iadd3_imad_mix_Gops": round(ap["mix"]["units_per_s"] / 1e9, 1),
                    "fp64_maxplus_cell_Gcells": round(ap["dcell"]["units_per_s"] / 1e9, 1),
                    "frac_of_mix": round(achieved / (ap["mix"]["units_per_s"] / 1e9), 4),
                    "cells_frac_of_fp64_cell_peak": round(cells / (my_ms / 1e3) / ap["dcell"]["units_per_s"], 4),
                    "from": "profiles/r02/alu_peak.json (B200, 1965 MHz)"}
    except (OSError, KeyError, ValueError):
        measured = None

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 1), "unit": "configs/s", "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": round(tot_ms / a.steps, 4), "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
                "config": {"workload": cfg["name"], "n_candidates": N, "k": a.k,
                           "step": "full sweep -> exact global top-k (one 1F1B run per distinct class pipeline, "
                                   "see `no_dedup`; gradient sync pruned where T0 already exceeds the top-k bound, "
                                   "see `unpruned`)",
                           "l2": "flushed between timed steps (512 MiB write, outside the event intervals)",
                           "parallelism": f"block-cyclic shard x{world}" + (" + NCCL all_gather" if world > 1 else "")},
                "roofline": {"bound": "alu", "achieved": round(achieved, 1), "peak": round(peak_gops, 1),
                             "unit": "Gop/s", "frac": round(achieved / peak_gops, 4), "traffic": traffic,
                             "issue_slots": issue, "ops_cells": OPS_PER_CELL * cells, "ops_overhead": over,
                             "kernel": "one hsim_topk sweep = K_split, K_pipe<P>, K_deep (concurrent fork/join "
                                       "streams), K_final with the pruned gradient sync, K_merge; per-kernel shares "
                                       "in profiles/",
                             "ops_per_launch": ops, "cells_per_launch": cells,
                             "peak_from": f"{SMS} SMs x {LANES_PER_SM} lanes x {sm_max:.0f} MHz (issue slots)",
                             "measured_peaks": measured},
                "gpu_launches": launches_per_step * a.steps,
                "clocks": clk}
        if e2e:
            line["e2e"] = e2e
        if e2e_sweep:
            line["e2e_sweep"] = e2e_sweep
        if unpruned:
            line["unpruned"] = unpruned
        if no_dedup:
            line["no_dedup"] = no_dedup
        if world == 1 and not a.no_cpu:
            line["cpu_baseline"] = cpu_baseline(cfg)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
