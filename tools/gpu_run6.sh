#!/bin/bash
# full GPU suite + bench + variant sweep timings
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=15 > gpurun_out/gputest6.log 2>&1; tail -22 gpurun_out/gputest6.log
python - > gpurun_out/variant_timing6.log 2>&1 <<'PY'
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
tm("config2 default", H.get(2))
tm("config2 interleave v=2", H.with_interleave(H.get(2), 2))
tm("config2 interleave v=4", H.with_interleave(H.get(2), 4))
tm("config4 default", H.get(4))
tm("config4 ep_dp", H.with_ep_dp(H.get(4)))
tm("config4 interleave v=2", H.with_interleave(H.get(4), 2))
tm("config3 interleave v=2", H.with_interleave(H.get(3), 2), reps=2)
PY
cat gpurun_out/variant_timing6.log
timeout 300 python bench.py --steps 100 --warmup 5 > gpurun_out/bench6.log 2>&1; tail -1 gpurun_out/bench6.log | cut -c1-400
