#!/bin/bash
# full GPU suite + bench on the current HEAD
mkdir -p gpurun_out
timeout 300 python bench.py --steps 100 --warmup 5 > gpurun_out/bench19.log 2>&1; tail -1 gpurun_out/bench19.log | cut -c1-300
timeout 1800 python -m pytest tests -m gpu -q -rs --durations=5 > gpurun_out/gputest19.log 2>&1; tail -10 gpurun_out/gputest19.log
