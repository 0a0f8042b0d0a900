#!/bin/bash
# Round-2 re-entry GPU call: full GPU suite (incl. f3), f3 timing, bench, launch list.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -rs --durations=20 > gpurun_out/gputest4.log 2>&1; tail -30 gpurun_out/gputest4.log
python - > gpurun_out/flow_timing.log 2>&1 <<'PY'
import time, torch, hsim_inputs as H
from paper_2508_05370_b200 import Sim
for n in (2, 4, 5):
    s = Sim(H.get(n)); _, top = s.topk(16); torch.cuda.synchronize()
    for rep in range(3):
        t = time.perf_counter(); out = s.flow_resim(top); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(n, f"{dt*1e3:.2f} ms for 16", out[:4].tolist())
PY
cat gpurun_out/flow_timing.log
timeout 300 python bench.py --steps 100 --warmup 5 > gpurun_out/bench4.log 2>&1; tail -2 gpurun_out/bench4.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench4_ref.log 2>&1; tail -1 gpurun_out/bench4_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches4.csv python bench.py --steps 2 --warmup 1 > gpurun_out/b_ncu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()"
