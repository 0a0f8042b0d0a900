#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_parity_gpu.py -q -k "pruned" > gpurun_out/prune20.log 2>&1; tail -2 gpurun_out/prune20.log
timeout 400 python bench.py --steps 100 --warmup 5 > gpurun_out/bench20.log 2>&1; tail -1 gpurun_out/bench20.log
