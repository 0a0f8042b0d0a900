#!/bin/bash
mkdir -p gpurun_out
for pr in 0 1; do
  for c in 2 4 3; do HSIM_PRUNE=$pr python tools/variant_bench.py $c 10 | sed "s/^/prune=$pr /"; done
done
HSIM_TRACE=1 python tools/trace_sweep.py 2 3 2> gpurun_out/trace13.log; grep -A30 "call 2" gpurun_out/trace13.log
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_parity_overlap_gpu.py tests/test_parity_gpu_r2.py tests/test_parity_variants_gpu.py -x -q > gpurun_out/parity13.log 2>&1; tail -4 gpurun_out/parity13.log
python - <<'PY'
import torch, hsim_inputs as H
from paper_2508_05370_b200 import Sim
def tm(name, cfg, reps=5):
    s = Sim(cfg); N = s.space_size()
    s.topk(16); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): s.topk(16)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{name}: N={N} {ms:.3f} ms/sweep {N / ms / 1e6:.3f} Gcand/s")
tm("config2 interleave v=2", H.with_interleave(H.get(2), 2))
tm("config2 interleave v=4", H.with_interleave(H.get(2), 4))
tm("config4 interleave v=2", H.with_interleave(H.get(4), 2))
tm("config3 interleave v=2", H.with_interleave(H.get(3), 2), reps=2)
tm("config2 overlap", H.with_sync_overlap(H.get(2)))
tm("config2 buckets+overlap", H.with_changes(H.with_sync_overlap(H.get(2)), search__sync_buckets=2))
PY
