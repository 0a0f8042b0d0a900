"""Command line: sweep one workload's candidate space on the GPU(s) and print
the best mappings.

  python -m paper_2508_05370_b200 --config 2 --k 5
  python -m paper_2508_05370_b200 --workload my_workload.json --mem-check
  torchrun --nproc-per-node 8 -m paper_2508_05370_b200 --config 5 --k 10

A workload is the dict of hsim_inputs.configs (cluster / model / search; the
JSON form is the same dict).  Each reported mapping is decoded on the host
(hsim_decode): micro-batch size, per class the stage device types and TP
degrees, layer split, micro-batches per replica and placement.
"""
import argparse
import json
import os
import sys


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_2508_05370_b200")
    g = ap.add_mutually_exclusive_group(required=True)
    g.add_argument("--config", type=int, help="BASELINE.json config 1-5 (hsim_inputs.configs)")
    g.add_argument("--workload", help="workload JSON file (the hsim_inputs dict form)")
    ap.add_argument("--k", type=int, default=5)
    ap.add_argument("--mem-check", action="store_true", help="prune mappings that do not fit (DESIGN.md M.1)")
    ap.add_argument("--sync-overlap", action="store_true", help="overlap the gradient sync (DESIGN.md S.1)")
    ap.add_argument("--json", action="store_true", help="print one JSON object instead of a table")
    a = ap.parse_args(argv)

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    import hsim_inputs as H
    from . import Sim, build
    from .sweep import sweep

    cfg = H.get(a.config) if a.config else json.load(open(a.workload))
    if a.mem_check:
        cfg = H.with_mem_check(cfg)
    if a.sync_overlap:
        cfg = H.with_sync_overlap(cfg)
    world = int(os.environ.get("WORLD_SIZE", 1))
    rank = int(os.environ.get("RANK", 0))
    if world > 1:
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()
    sim = Sim(cfg)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t, i = sweep(sim, a.k)
    e1.record()
    torch.cuda.synchronize()
    if rank == 0:
        N = sim.space_size()
        rows = [{"rank": r, "index": int(ii), "t_iter_ns": int(tt), "plan": sim.decode(int(ii))}
                for r, (tt, ii) in enumerate(zip(t.cpu().tolist(), i.cpu().tolist())) if ii >= 0]
        if a.json:
            print(json.dumps({"workload": cfg.get("name"), "candidates": N, "gpus": world,
                              "sweep_ms": e0.elapsed_time(e1), "top": rows}))
        else:
            print(f"{cfg.get('name')}: {N} candidates on {world} GPU(s), sweep {e0.elapsed_time(e1):.2f} ms")
            for row in rows:
                p = row["plan"]
                cls = "; ".join(
                    f"D={c['D']} stages(type,tp)={c['stages']} layers={c['layers']}" for c in p["classes"])
                print(f"#{row['rank'] + 1}  T_iter = {row['t_iter_ns'] / 1e6:.3f} ms  index {row['index']}  "
                      f"b={p['b']}  {cls}")
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
