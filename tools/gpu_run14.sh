#!/bin/bash
mkdir -p gpurun_out
for pr in 0 1 0 1; do HSIM_PRUNE=$pr timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prune=$pr', d['ms_per_step'], d['value'])"; done
HSIM_PRUNE=0 HSIM_TRACE=1 python tools/trace_sweep.py 2 3 2> gpurun_out/trace14a.log; grep -A30 "call 2" gpurun_out/trace14a.log
timeout 1500 python -m pytest tests/test_parity_gpu.py tests/test_parity_overlap_gpu.py tests/test_parity_gpu_r2.py tests/test_parity_variants_gpu.py tests/test_parity_memcheck_gpu.py -x -q > gpurun_out/parity14.log 2>&1; tail -4 gpurun_out/parity14.log
