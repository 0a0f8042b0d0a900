#!/bin/bash
# Round-2 GPU call: full GPU test suite, ALU microbenchmarks, sanitizers, bench.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
python tools/alu_peak.py --ncu > gpurun_out/alu_peak.log 2>&1; cp profiles/alu_peak_r02.json gpurun_out/ 2>/dev/null
timeout 1200 python -m pytest tests -m gpu -q -rs --durations=15 > gpurun_out/gputest2.log 2>&1; tail -25 gpurun_out/gputest2.log
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_run.py small > gpurun_out/cs_$t.log 2>&1; tail -4 gpurun_out/cs_$t.log
done
timeout 300 python bench.py --steps 100 --warmup 5 > gpurun_out/bench2.log 2>&1; tail -2 gpurun_out/bench2.log
