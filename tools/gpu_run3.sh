#!/bin/bash
# f3 GPU parity + source-level ncu captures of the sweep's main kernels.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_flow_gpu.py -x -q > gpurun_out/flowtest.log 2>&1; tail -15 gpurun_out/flowtest.log
python - > gpurun_out/flow_timing.log 2>&1 <<'PY'
import time, torch, hsim_inputs as H
from paper_2508_05370_b200 import Sim
for n in (2, 4, 5):
    s = Sim(H.get(n)); _, top = s.topk(16); torch.cuda.synchronize()
    for rep in range(2):
        t = time.perf_counter(); out = s.flow_resim(top); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(n, f"{dt*1e3:.2f} ms for 16", out[:4].tolist())
PY
cat gpurun_out/flow_timing.log
for k in k_sync k_split k_final_small; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"^${k}" -s 1 -c 1 -o gpurun_out/prof_$k python tools/prof_sweep.py 2 2 > /dev/null 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_pipe" --kernel-name-base demangled -s 2 -c 1 -o gpurun_out/prof_pipe python tools/prof_sweep.py 2 2 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
